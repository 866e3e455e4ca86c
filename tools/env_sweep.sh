#!/bin/bash
# Bench under several environment settings (graph mode): tools/env_sweep.sh <tag> "<ENV=V ...>" ...
set -u
tag=$1; shift
out=gpurun_out/$tag; mkdir -p "$out"
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs python bench.py --no-sweep --no-e2e --gs-steps 2 --steps 20 > "$out/sweep$i.json" 2> "$out/sweep$i.err"
  python - "$out/sweep$i.json" "$envs" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
g = d.get("gs", {})
print(f"[{sys.argv[2]}] OSPR {d['value']:.0f} sf/s ({d['ms_per_step']*1e3:.1f} us)  GS {g.get('value', 0):.0f} it/s",
      {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()},
      {k: round(v['avg_us'], 1) for k, v in g.get('kernels', {}).items()})
PY
done
