mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/graph_cond scripts/micro/graph_cond.cu > gpurun_out/micro.log 2>&1
timeout 60 /tmp/graph_cond >> gpurun_out/micro.log 2>&1; echo "micro rc=$?" >> gpurun_out/micro.log
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1700 python -m pytest tests/test_gpu_graph.py tests/test_gpu_edges.py tests/test_gpu_production_kernels.py tests/test_gpu_parity.py -m gpu -q -rf --timeout 600 > gpurun_out/pytest_g2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_g2.log
tail -30 gpurun_out/pytest_g2.log; cat gpurun_out/micro.log
