#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full capture.
# usage: scripts/gpu_round.sh [tag]
#   NCU=launch (default) runs the launch-list pass, NCU=full the one full capture (without the
#   tests/bench: one profiler tool per call), NCU=0 none.
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
if [ "${NCU:-launch}" != "full" ]; then
timeout 1200 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
if [ "${NCU:-launch}" = "launch" ]; then
  timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
      --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
elif [ "${NCU}" = "full" ]; then
  timeout 600 $CMD > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k_sweep2t_col|k_spmv_tma|k_restrict_black_xyz|k_prolong_black4|k_axpy_norm|k_sweep_col|k_resid_restrict_col|k_tailsm" -s 0 -c 40 \
      -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
fi
