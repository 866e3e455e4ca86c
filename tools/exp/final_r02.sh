#!/bin/bash
# Round-2 validation and evidence: GPU tests, smoke, full bench line, warm launch list, ncu --set full
# of the OSPR kernels at C3 and C5 and of the GS passes at C4 size.
set -u
out=gpurun_out/${1:-r02_final}; mkdir -p "$out"
nvidia-smi > "$out/nvidia-smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"; tail -2 "$out/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; echo "smoke rc=$?"; tail -1 "$out/smoke.log"
timeout 900 python bench.py > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --gs-steps 1 > "$out/bench_small.json" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file "$out/launches_warm.csv" python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --gs-steps 1 \
    > "$out/ncu_launches.log" 2>&1
echo "ncu launches rc=$?"
python tools/prof_run.py ospr 3 > "$out/ospr_plain.log" 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ospr_rows_a2|col_pipe|ospr_rows_cf" -s 3 -c 3 \
    -o "$out/ospr" python tools/prof_run.py ospr 3 > "$out/ncu_ospr.log" 2>&1
echo "ncu ospr rc=$?"
python tools/prof_run.py c5 2 > "$out/c5_plain.log" 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ospr_rows_a2|col_pipe_g2|ospr_rows_cf" -s 3 -c 3 \
    -o "$out/c5" python tools/prof_run.py c5 2 > "$out/ncu_c5.log" 2>&1
echo "ncu c5 rc=$?"
python tools/prof_run.py gs64 1 > "$out/gs_plain.log" 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:col_pipe|gs_rows_kernel" -s 2 -c 2 \
    -o "$out/gs64" python tools/prof_run.py gs64 1 > "$out/ncu_gs.log" 2>&1
echo "ncu gs rc=$?"
# summaries on the box (the .ncu-rep files exceed what gpurun copies back), then drop the reports
for r in ospr c5 gs64; do
    [ -f "$out/$r.ncu-rep" ] || continue
    python tools/ncu_summary.py "$out/$r.ncu-rep" --src 12 > "$out/ncu_${r}_summary.txt" 2>&1
    ncu -i "$out/$r.ncu-rep" --page raw --csv > "$out/ncu_${r}_raw.csv" 2>/dev/null
done
cp profiles/ncu_traffic.json "$out/ncu_traffic_before.json"
[ -f "$out/ospr.ncu-rep" ] && python tools/ncu_traffic.py "$out/ospr.ncu-rep" "ncu --set full --clock-control none (caches flushed per replay); OSPR classes: tools/prof_run.py ospr 3 (C3 OSPR call, 12 pairs, L=2^16), capture ${1:-r02_final}/ospr" > /dev/null
[ -f "$out/gs64.ncu-rep" ] && python tools/ncu_traffic.py "$out/gs64.ncu-rep" "gs_cols/gs_rows: tools/prof_run.py gs64 1 (the whole C4 launch group: 64 frames, 512 MiB state streaming from HBM), capture ${1:-r02_final}/gs64" --merge > /dev/null
cp profiles/ncu_traffic.json "$out/ncu_traffic.json"
rm -f "$out"/*.ncu-rep
ls -la "$out"
