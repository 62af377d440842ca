# r02i: fused triples of half-sweeps (k_sweep3t_col): correctness forced on small levels, bench A/B
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
MSS_TRIPLE=2 MSS_PAIR=1 MSS_PAIR_TY=16 timeout 900 python -m pytest tests/test_gpu_production_kernels.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "not nccl" > gpurun_out/pytest_triple_forced.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_triple_forced.log
tail -15 gpurun_out/pytest_triple_forced.log
for t in 1 0; do
  MSS_TRIPLE=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_t$t.log 2>&1
done
python - <<'PY'
import json
for t in (1, 0):
    try:
        d = json.loads([l for l in open(f"gpurun_out/bench_t{t}.log") if l.startswith("{")][-1])
        print(t, d["value"], d["ms_per_step"], d["config"]["iters_per_level"], d["config"]["true_rel_res"], d["level_split"])
        print({k: v for k, v in d["kernels"].items() if "@L0" in k})
    except Exception as e:
        print(t, "ERR", e, open(f"gpurun_out/bench_t{t}.log").read()[-2000:])
PY
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
tail -5 gpurun_out/pytest_full.log
