mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_graph.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --control host > gpurun_out/bench_host.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -rf --timeout 900 > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
tail -5 gpurun_out/pytest_full.log
python - <<'PY'
import json
for f in ["gpurun_out/bench_graph.log","gpurun_out/bench_host.log"]:
    try:
        d=json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f, d["value"], d["ms_per_step"], d.get("control"), d.get("setup_ms"), d.get("setup_coarsest_ms"), d["roofline"]["frac"], d["gpu_launches"], d.get("level_split"))
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-2000:])
PY
