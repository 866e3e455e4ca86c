#!/bin/bash
# ncu launch list of the bench command (per-launch device time; warm caches, serialised):
# tools/launch_list.sh <tag> [bench args...]
set -u
tag=$1; shift
out=gpurun_out/$tag; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py "$@" > "$out/plain.json" 2> "$out/plain.err" && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file "$out/launches.csv" python bench.py "$@" > "$out/ncu.log" 2>&1
echo "rc=$?"
python tools/launch_summary.py "$out/launches.csv" | head -20
