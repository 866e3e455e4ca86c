#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list and one
# full capture of the named kernels.  usage: tools/gpu_round.sh <tag> [kernel-regex] [tests]
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh r01 "ospr_cols|gs_cols"'
set -u
tag=${1:-run}
kre=${2:-"ospr_cols|gs_cols"}
tests=${3:-1}
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi > "$out/nvidia-smi.txt" 2>&1
lscpu > "$out/lscpu.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; exit 1; }
if [ "$tests" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1
  echo "pytest gpu rc=$?" ; tail -3 "$out/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1
  echo "smoke rc=$?"; tail -2 "$out/smoke.log"
fi
timeout 900 python bench.py > "$out/bench.json" 2> "$out/bench.err"
echo "bench rc=$?"; cut -c1-600 "$out/bench.json"
# launch list (cold-cache, serialised) of the bench's OSPR+GS step at reduced K
timeout 600 python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --gs-steps 1 > "$out/bench_small.json" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$out/launches.csv" python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --gs-steps 1 \
    > "$out/ncu_launches.log" 2>&1
echo "ncu launches rc=$?"
timeout 300 python tools/prof_run.py all 3 > "$out/prof_plain.log" 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 4 \
    -o "$out/prof" python tools/prof_run.py all 3 > "$out/ncu_full.log" 2>&1
echo "ncu full rc=$?"
ls -la "$out"
