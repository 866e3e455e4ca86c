#!/bin/bash
# Copy a validation run's evidence (tools/exp/final_r02.sh <name>) into profiles/.
set -eu
d=gpurun_out/${1:?run name}
cp "$d/bench.json" profiles/r02_bench_latest.json
python tools/launch_summary.py "$d/launches_warm.csv" > profiles/r02_launches_warm.txt
cp "$d/ncu_ospr_summary.txt" profiles/r02_ncu_ospr_c3.txt
cp "$d/ncu_c5_summary.txt" profiles/r02_ncu_ospr_c5.txt
cp "$d/ncu_gs64_summary.txt" profiles/r02_ncu_gs_c4_64frames.txt
cp "$d/ncu_traffic.json" profiles/ncu_traffic.json
cp "$d/launches_warm.csv" profiles/r02_launches_warm.csv
