#!/bin/bash
# Sweep env-selected kernel variants on C5 (diagnostic; prints probe.py breakdowns).
# usage: PROBE_ARGS="--stream" scripts/gpu_variants.sh "ENV=1 ENV2=3" "ENV=2" ...
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
( for v in "$@"; do
    echo "=== $v"; env $v timeout 300 python scripts/probe.py --config ${PROBE_CONFIG:-C5} --reps 2 --prof-level ${PROBE_LEVEL:-0} $PROBE_ARGS | head -${PROBE_LINES:-8}; done ) > gpurun_out/variants.log 2>&1
