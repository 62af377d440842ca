# r02d: branch-free 3-D tail passes; events fix; C4 chain exploration (explicit level_dims)
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_d.log 2>&1
i=0
for ld in '[[128,128,128],[32,32,128],[16,16,32],[4,4,16]]' '[[128,128,128],[64,64,128],[16,16,32]]' '[[128,128,128],[64,64,128],[16,16,32],[4,4,8]]' '[[128,128,128],[32,32,128],[8,8,32]]' '[[128,128,128],[32,32,128],[16,16,32]]' '[[128,128,128],[64,64,128],[32,32,32],[8,8,8]]'; do
  i=$((i+1))
  timeout 300 python scripts/probe.py --config C4 --reps 3 --params "{\"level_dims\": $ld}" > gpurun_out/probe_C4_chain$i.log 2>&1
done
timeout 300 python scripts/probe.py --config C4 --reps 3 --params '{"dims_mode": 4}' > gpurun_out/probe_C4_dm4.log 2>&1
timeout 300 python scripts/probe.py --config C4 --reps 3 > gpurun_out/probe_C4_dm0.log 2>&1
timeout 300 python scripts/probe.py --config C2 --reps 5 > gpurun_out/probe_C2.log 2>&1
timeout 1500 python -m pytest tests/ -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/bench_d.log") if l.startswith("{")][-1])
print(d["value"], d["ms_per_step"], d["level_split"], d["kernels"]["tail@L2"])
PY
for f in gpurun_out/probe_C*.log; do echo "== $f"; head -3 $f; done
