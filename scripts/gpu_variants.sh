#!/bin/bash
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
( for v in "MSS_COL_MINB=3" "MSS_COL_MINB=4" "MSS_COL_MINB=5" "MSS_COL_MINB=4 MSS_COL_NCH=4" "MSS_COL_MINB=4 MSS_COL_NCH=16" "MSS_COL_MINB=5 MSS_COL_NCH=16" "MSS_NO_COLWALK=1"; do
    echo "=== $v"; env $v timeout 300 python scripts/probe.py --config C5 --reps 2 --prof-level 0 | head -8; done ) > gpurun_out/variants.log 2>&1
