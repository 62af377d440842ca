# r02e: full GPU suite (no -x) + ncu source-level capture of the cluster tail
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/probe.py --config C5 --reps 2 > gpurun_out/probe_C5_e.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tailsm -s 20 -c 1 -o gpurun_out/r02e_tail -f python scripts/probe.py --config C5 --reps 1 > gpurun_out/ncu_tail.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_tail.log
timeout 2000 python -m pytest tests/ -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -8 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/ncu_tail.log; head -3 gpurun_out/probe_C5_e.log
