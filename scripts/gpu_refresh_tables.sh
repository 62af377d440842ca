#!/bin/bash
# Re-measure the N-scaling table and the comparison-methods table of DESIGN.md §9 (probe.py).
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
( for n in 64 128 256 384 512; do timeout 300 python scripts/probe.py --config C5 --n $n --reps 3 --prof-level -1 | sed -n 1,2p; done ) > gpurun_out/n_scaling.log 2>&1
( for c in C5 C4 C2; do for m in 0 1 3; do echo "== $c method $m"; timeout 300 python scripts/probe.py --config $c --reps 3 --prof-level -1 --params "{\"method\": $m}" | sed -n 1,2p; done; done ) > gpurun_out/methods.log 2>&1
