mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_production_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -rf --timeout 900 -x > gpurun_out/pytest_new.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_new.log
tail -5 gpurun_out/pytest_new.log
