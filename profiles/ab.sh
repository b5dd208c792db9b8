#!/usr/bin/env bash
# A/B of build knobs on the GPU box: for each KNOBS variant (-D build knobs, device and host), rebuild _prx.so in-tree and run
# the C4 bench; prints one "variant ms_per_step stages" line each.  The last variant built is
# left in place, so list the default last.
#   usage: bash profiles/ab.sh "-DPRX_VERTEX_SOA=0" ""
set -uo pipefail
mkdir -p gpurun_out
for v in "$@"; do
    make -s -C paper_2111_06906_b200 clean >/dev/null
    make -s -j 16 -C paper_2111_06906_b200 KNOBS="$v" >/dev/null 2>gpurun_out/ab_build.err || { echo "build failed: $v"; tail gpurun_out/ab_build.err; continue; }
    for rep in 1 2; do
        python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-splat-sweep ${BENCH_ARGS:-} 2>/dev/null \
          | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant [$v] rep $rep:', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['stages_ms'].items()})"
    done
done
