#!/bin/bash
# quick perf probe: tests, C5/C4/C2 breakdown, optional ncu of the level-0 kernels
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
( for c in "C5" "C4" "C2"; do timeout 300 python scripts/probe.py --config $c; done;
  MSS_NO_COLWALK=1 timeout 300 python scripts/probe.py --config C5 ) > gpurun_out/probe.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
  P="python scripts/probe.py --config C5 --reps 1"
  timeout 300 $P > gpurun_out/plain_l0.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
     -k regex:"k_sweep_col|k_spmv_col|k_resid_restrict|k_prolong_black|k_axpy_norm" \
     -s 0 -c 12 -o gpurun_out/prof_l0c $P > gpurun_out/ncu_l0.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_l0.log
fi
