#!/bin/bash
# Diagnostic GPU session: tests, probes per config, ncu of the tail and level-0 sweep.
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
( for c in "C5 --n 128" "C2" "C4" "C3 --params {\"use_lift\":0,\"interp\":1}" "C5"; do
    timeout 300 python scripts/probe.py --config $c; done ) > gpurun_out/probe.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
  P="python scripts/probe.py --config C5 --n 128 --reps 1"
  timeout 300 $P > gpurun_out/plain_tail.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 2 -c 1 \
      -o gpurun_out/prof_tail $P > gpurun_out/ncu_tail.log 2>&1
  echo "ncu tail rc=$?" >> gpurun_out/ncu_tail.log
  P="python scripts/probe.py --config C5 --reps 1"
  timeout 300 $P > gpurun_out/plain_l0.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_halfsweep|k_pdir|k_resid_restrict|k_prolong_black|k_axpy_norm" -s 0 -c 8 \
      -o gpurun_out/prof_l0 $P > gpurun_out/ncu_l0.log 2>&1
  echo "ncu l0 rc=$?" >> gpurun_out/ncu_l0.log
fi
