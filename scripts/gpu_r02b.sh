# r02b: L2 residency of the level-1 sweep operands (A/B) and the batched-load cluster tail
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
for mb in 96 0; do
  MSS_L2KEEP_MB=$mb timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_l2_$mb.log 2>&1
done
for c in C4 C2; do
  for mb in 96 0; do
    MSS_L2KEEP_MB=$mb timeout 120 python scripts/probe.py --config $c --reps 5 > gpurun_out/probe_${c}_$mb.log 2>&1
  done
done
MSS_TAIL_PHASES=1 timeout 120 python scripts/probe.py --config C5 --reps 2 > gpurun_out/probe_C5_phases.log 2>&1
timeout 1500 python -m pytest tests/ -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python - <<'PY'
import json
for mb in (96, 0):
    f = f"gpurun_out/bench_l2_{mb}.log"
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f, d["value"], d["ms_per_step"], d["level_split"], {k: v["ms"] for k, v in d["kernels"].items() if "@L1" in k or "tail" in k})
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-1500:])
PY
for f in gpurun_out/probe_*.log; do echo "== $f"; tail -12 $f; done
