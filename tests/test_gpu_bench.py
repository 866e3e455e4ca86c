"""bench.py keeps the driver's JSON contract on a B200 (a short run: C3 headline + e2e; the
sweep, GS and C5 blocks off): one line, the headline metric and unit, roofline, cpu_baseline,
e2e with the host-copy byte counts, gpu_launches and the clocks sampled during the timed region."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--no-sweep",
                        "--no-gs", "--no-c5"], capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["unit"] == "sub-frames/s" and d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert "workload" in d["config"] and "l2" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 1024 * 1024 * 4            # the C3 target, fp32
    assert e["d2h_bytes_per_step"] == 24 * 1024 * 128 + 8        # packed holograms + the MSE
    assert d["gpu_launches"] >= 3 * 4                             # a0 + three passes per step
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


@pytest.mark.parametrize("env,args,key", [
    ({"HOLO_BENCH_FAKE_WORLD": "4"}, ["--no-c5", "--no-e2e"], None),          # C3 split over 4 "ranks"
    ({"HOLO_BENCH_FAKE_SHARDS": "4"}, ["--no-e2e"], "c5_video"),              # C5 video, 4-way shards
])
def test_bench_sharded_step_structures(env, args, key):
    """The N > 1 step structures (sub-frame shards, the exchange around the graphed shard, the
    video pipeline's side stream) run on one GPU with stand-in collectives (testing hooks of
    bench.py); the line stays well formed."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--no-sweep",
                        "--no-gs"] + args, capture_output=True, text=True, cwd=ROOT, timeout=900,
                       env=dict(os.environ, **env))
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")][-1])
    assert d["value"] > 0
    if key:
        v = d[key]
        assert v["value"] > 0 and "FAKE" in v["config"]["partition"]
        assert v["shard"]["sub_frames"][1] - v["shard"]["sub_frames"][0] == 8     # 32 sub-frames / 4
    else:
        assert "sub-frame shards x4" in d["config"]["parallelism"]
