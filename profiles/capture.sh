#!/usr/bin/env bash
# Profiling recipe run on the GPU box (see /opt/skills/guides/B200_PROFILING.md):
#   1. the plain bench (must exit 0 before any ncu pass),
#   2. the launch list of the same command (cold-cache, serialised per-launch times),
#   3. `ncu --set full` of one steady-state launch of each hot kernel (4th launch: frame 3),
#      one ncu process per kernel so --launch-skip counts that kernel alone,
#   4. the same for the atomic splat's kernels (bench --splat-mode 0).
# Outputs land in gpurun_out/; profiles/summarize.py turns them into profiles/TAG_*.
set -uo pipefail
tag=${1:-r02}
out=gpurun_out
mkdir -p "$out"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > "$out/${tag}_bench.json" 2> "$out/${tag}_bench.err" || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/${tag}_launches.csv" \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-splat-sweep --extra none --splat-overlap 0 > "$out/${tag}_ncu_launches.log" 2>&1
common="--set full --import-source on --clock-control none"
# (ncu serialises kernels, so the overlapped splat has nothing to overlap under it: the launch
# list and the captures use the serial loop, whose frames list each splat after its frame)
bench="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-splat-sweep --extra none --splat-overlap 0"
for k in k_trace k_verify_error_walk k_occlusion_flags k_compute_dm k_gather_bin k_gather_staged \
         k_rs_scatter k_fill_assign k_update_origins; do
    skip=3
    [ "$k" = k_rs_scatter ] && skip=18   # 5 radix passes per frame (3 prune + 2 gather: 18 = frame 3's first gather pass)
    [ "$k" = k_fill_assign ] && skip=6   # one per light
    case "$k" in k_verify_error_walk|k_occlusion_flags|k_update_origins) skip=2 ;; esac  # from frame 1 on
    ncu $common -k "regex:${k}(<|$)" --launch-skip $skip -c 1 -o "$out/${tag}_full_${k}" $bench \
        > "$out/${tag}_ncu_${k}.log" 2>&1 || echo "ncu $k rc=$?"
done
for k in k_bin_filter k_bin_scatter k_splat_pixels; do
    ncu $common -k "regex:${k}(<|$)" --launch-skip 3 -c 1 -o "$out/${tag}_full_${k}" $bench --splat-mode 0 \
        > "$out/${tag}_ncu_${k}.log" 2>&1 || echo "ncu $k rc=$?"
done
ls -la "$out"
