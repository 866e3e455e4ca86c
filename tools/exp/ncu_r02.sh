#!/bin/bash
# Round-2 ncu evidence: --set full of the OSPR kernels (C3) and of the GS passes at C4 size
# (64 frames, 512 MiB state), plus the warm launch list of the bench step.
set -u
out=gpurun_out/${1:-r02_ncu}; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; exit 1; }
python tools/prof_run.py ospr 3 > "$out/ospr_plain.log" 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ospr_rows_a2|col_pipe|ospr_rows_cf" -s 3 -c 3 \
    -o "$out/ospr" python tools/prof_run.py ospr 3 > "$out/ncu_ospr.log" 2>&1
echo "ncu ospr rc=$?"
python tools/prof_run.py gs64 1 > "$out/gs_plain.log" 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:col_pipe|gs_rows_kernel" -s 2 -c 2 \
    -o "$out/gs64" python tools/prof_run.py gs64 1 > "$out/ncu_gs.log" 2>&1
echo "ncu gs rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --gs-steps 1 > "$out/bench_small.json" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file "$out/launches_warm.csv" python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --gs-steps 1 \
    > "$out/ncu_launches.log" 2>&1
echo "ncu launches rc=$?"
ls -la "$out"
