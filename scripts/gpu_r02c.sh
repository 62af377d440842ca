# r02c: level-tree events + automatic semi-coarsening parity; C4 with the aspect chain
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_events.py tests/test_gpu_semicoarsening.py -m gpu -q -rf --timeout 600 -s > gpurun_out/pytest_new.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_new.log
for dm in 0 3; do
  timeout 300 python scripts/probe.py --config C4 --reps 5 --params "{\"dims_mode\": $dm}" > gpurun_out/probe_C4_dm$dm.log 2>&1
done
timeout 300 python scripts/probe.py --config C4 --reps 5 --params '{"level_dims": [[128,128,128],[64,64,128],[16,16,32]]}' > gpurun_out/probe_C4_explicit.log 2>&1
tail -5 gpurun_out/pytest_new.log
for f in gpurun_out/probe_C4_*.log; do echo "== $f"; head -4 $f; done
