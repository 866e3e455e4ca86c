#!/bin/bash
# GS normalisation variants: drift vs the oracle (+ numpy complex64 control) and GS speed.
set -u
out=gpurun_out/${1:-r02_gsvar}; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; tail "$out/build.log"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gs.py -x -q > "$out/pytest_gs.log" 2>&1; echo "pytest rc=$?"; tail -5 "$out/pytest_gs.log"
for v in product r01 norm0 norm2; do
  lib=tools/exp/libholo_$v.so; [ $v = product ] && lib=paper_2004_04049_b200/libholo.so
  timeout 600 python tools/gs_drift.py "$out/drift_$v.json" --lib $lib > "$out/drift_$v.log" 2>&1; echo "== $v drift rc=$?"; grep -v "^   it" "$out/drift_$v.log" | tail -6
  timeout 300 python tools/with_lib.py $lib bench.py --no-sweep --no-e2e --no-c5 --steps 5 --gs-steps 3 > "$out/bench_$v.json" 2> "$out/bench_$v.err"
  python - "$out/bench_$v.json" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); g=d["gs"]
print("  GS", round(g["value"]), "it/s", {k: round(v["avg_us"],1) for k,v in g["kernels"].items()})
PY
done
