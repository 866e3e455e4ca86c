#!/bin/bash
# OSPR chunk-budget sweep (tooling): C3 and C5 bench values under HOLO_OSPR_CHUNK_BYTES settings.
for e in "HOLO_X=0" "HOLO_OSPR_CHUNK_BYTES=201326592" "HOLO_OSPR_CHUNK_BYTES=536870912"; do
  env $e timeout 600 python bench.py --no-sweep --no-gs --no-e2e > gpurun_out/c5_$$.json 2>/dev/null
  python - "$e" gpurun_out/c5_$$.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], "C3", round(d["value"]), "C5", round(d["c5"]["value"]), round(d["c5"]["ms_per_step"],3))
PY
done
