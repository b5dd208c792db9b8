#!/usr/bin/env bash
# Profiling recipe run on the GPU box (see /opt/skills/guides/B200_PROFILING.md):
#   1. the plain bench (must exit 0 before any ncu pass),
#   2. the launch list of the same command (cold-cache, serialised per-launch times),
#   3. one `ncu --set full` capture of the hot traversal kernels of a steady-state frame.
# Outputs land in gpurun_out/; summaries worth keeping are copied into profiles/.
set -euo pipefail
tag=${1:-r01}
out=gpurun_out
mkdir -p "$out"
python bench.py --steps 5 --warmup 3 > "$out/${tag}_bench.json" 2> "$out/${tag}_bench.err"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/${tag}_launches.csv" \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > "$out/${tag}_ncu_launches.log" 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"k_trace|k_verify_error_walk|k_gather_pixels|k_occlusion_flags" --launch-skip 7 -c 3 \
    -o "$out/${tag}_full" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > "$out/${tag}_ncu_full.log" 2>&1
