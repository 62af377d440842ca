# r02h: fused x+y restriction of the fused residual (A/B MSS_RESTRICT_XY)
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
for xy in 1 0; do
  MSS_RESTRICT_XY=$xy timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_xy$xy.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_production_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q --timeout 900 > gpurun_out/pytest_h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_h.log
tail -4 gpurun_out/pytest_h.log
python - <<'PY'
import json
for xy in (1, 0):
    d = json.loads([l for l in open(f"gpurun_out/bench_xy{xy}.log") if l.startswith("{")][-1])
    print(xy, d["value"], d["ms_per_step"], d["level_split"], d["kernels"]["restrict@L0"], d["kernels"].get("residual@L0"))
PY
