"""A/B timing of libholo variants through bench.py (GPU box): each variant is
`name[:lib.so][:ENV=V,ENV=V]`, run round-robin `--reps` times; prints the OSPR/GS/C5
values and the per-kernel times of each run.
usage: python tools/ab.py [--reps 2] [--bench "--no-sweep --no-e2e --no-gs"] v1 v2 ..."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--bench", default="--no-sweep --no-e2e --no-gs --no-c5 --steps 20")
ap.add_argument("variants", nargs="+")
a = ap.parse_args()
for rep in range(a.reps):
    for v in a.variants:
        f = v.split(":")
        name, lib = f[0], (f[1] if len(f) > 1 and f[1] else None)
        env = dict(os.environ)
        if len(f) > 2 and f[2]:
            for kv in f[2].split(","):
                k, val = kv.split("=", 1)
                env[k] = val
        cmd = [sys.executable] + ([os.path.join(ROOT, "tools/with_lib.py"), lib] if lib else []) + \
              [os.path.join(ROOT, "bench.py")] + a.bench.split()
        r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(f"[{name}] FAILED rc={r.returncode}\n{r.stderr[-2000:]}")
            continue
        out = f"[{name}] OSPR {d['value']:.0f} ({d['ms_per_step'] * 1e3:.1f} us) " + \
              " ".join(f"{k}={x['avg_us']:.1f}" for k, x in d.get("kernels", {}).items())
        if "gs" in d:
            out += f" | GS {d['gs']['value']:.0f} " + " ".join(f"{k}={x['avg_us']:.1f}" for k, x in d["gs"]["kernels"].items())
        if "c5" in d:
            out += f" | C5 {d['c5']['value']:.0f} ({d['c5']['ms_per_step'] * 1e3:.1f} us)"
        print(out, flush=True)
