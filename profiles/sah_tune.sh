#!/usr/bin/env bash
# SAH build knob sweep (C4 frame ms; device time). usage: bash profiles/sah_tune.sh
for cfg in "16 1.0 8" "32 1.0 8" "16 0.5 8" "16 2.0 8" "16 1.0 4" "32 2.0 8" "16 3.0 8"; do
  set -- $cfg
  PRX_SAH_BINS=$1 PRX_SAH_TRAV=$2 PRX_SAH_MAXLEAF=$3 timeout -s ABRT 300 python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('bins=$1 trav=$2 leaf=$3', round(d['ms_per_step'],3), 'verify', round(s['verify'],3), 'trace', round(s['trace'],3))"
done
