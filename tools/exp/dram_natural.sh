#!/bin/bash
# DRAM bytes per kernel in the bench's natural cache state (application replay, no cache control):
# tools/exp/dram_natural.sh <tag> [bench args]
set -u
tag=$1; shift
out=gpurun_out/$tag; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py "$@" > "$out/plain.json" 2> "$out/plain.err" || { echo bench failed; tail "$out/plain.err"; exit 1; }
timeout 1800 ncu --replay-mode application --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum \
  --csv --log-file "$out/natural.csv" python bench.py "$@" > "$out/ncu.log" 2>&1
echo "ncu rc=$?"; tail -3 "$out/ncu.log"
