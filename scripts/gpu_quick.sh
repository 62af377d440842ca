#!/bin/bash
# quick perf probe: C5 and C4 breakdown + ncu of the level-0 kernels (one of each)
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
( for c in "C5" "C4" "C2"; do timeout 300 python scripts/probe.py --config $c; done ) > gpurun_out/probe.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ "${NCU:-1}" = "1" ]; then
  P="python scripts/probe.py --config C5 --reps 1"
  timeout 300 $P > gpurun_out/plain_l0.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
     -k regex:"k_halfsweep<3, 0, 0>|k_halfsweep<3, 0, 1>|k_halfsweep<3, 1, 0>|k_pdir|k_resid_restrict|k_prolong_black|k_axpy_norm|k_restrict_axis" \
     -s 0 -c 40 -o gpurun_out/prof_l0b $P > gpurun_out/ncu_l0.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_l0.log
fi
