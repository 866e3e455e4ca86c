#!/bin/bash
# Quick GPU check: build, parity tests, bench (no sweep).  usage: tools/gpu_quick.sh <tag> [pytest -k expr] [bench args]
set -u
tag=$1; kexpr=${2:-}; shift 2 || true
out=gpurun_out/$tag; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; tail "$out/build.log"; exit 1; }
if [ "$kexpr" != "none" ]; then
  if [ -n "$kexpr" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "$kexpr" > "$out/pytest_gpu.log" 2>&1
  else timeout 1200 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1; fi
  echo "pytest rc=$?"; tail -15 "$out/pytest_gpu.log"
fi
timeout 600 python bench.py --no-sweep "$@" > "$out/bench.json" 2> "$out/bench.err"
echo "bench rc=$?"; tail -3 "$out/bench.err"
python - "$out/bench.json" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("OSPR", round(d["value"]), "sf/s", "ms/step", round(d["ms_per_step"],4), "e2e", round(d.get("e2e",{}).get("value",0)), "clk", d["clocks"])
print("roofline", {k: d["roofline"][k] for k in ("kernel","achieved","frac","avg_launch_us")})
for k,v in d["kernels"].items(): print("  ", k, round(v["avg_us"],2))
if "gs" in d:
    g=d["gs"]; print("GS", round(g["value"]), "it/s", {k: round(v["avg_us"],2) for k,v in g["kernels"].items()})
PY
