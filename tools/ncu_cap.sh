#!/bin/bash
# One ncu --set full capture: tools/ncu_cap.sh <tag> <kernel-regex> <skip> <count> <prof_run args...>
set -u
tag=$1; kre=$2; skip=$3; cnt=$4; shift 4
out=gpurun_out/$tag; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; exit 1; }
timeout 300 python tools/prof_run.py "$@" > "$out/prof_plain.log" 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c "$cnt" \
    -o "$out/prof" python tools/prof_run.py "$@" > "$out/ncu_full.log" 2>&1
echo "ncu rc=$?"; tail -3 "$out/ncu_full.log"
