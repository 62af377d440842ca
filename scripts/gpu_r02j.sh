# r02j: colour-split storage of the compile-time-dims tail level (A/B MSS_TAIL_CT)
mkdir -p gpurun_out
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
for ct in 1 0; do
  MSS_TAIL_CT=$ct MSS_TAIL_PHASES=1 timeout 300 python scripts/probe.py --config C5 --reps 3 > gpurun_out/probe_C5_ct$ct.log 2>&1
  MSS_TAIL_CT=$ct timeout 300 python scripts/probe.py --config C2 --reps 5 > gpurun_out/probe_C2_ct$ct.log 2>&1
  MSS_TAIL_CT=$ct timeout 300 python scripts/probe.py --config C4 --reps 3 > gpurun_out/probe_C4_ct$ct.log 2>&1
done
timeout 2000 python -m pytest tests/ -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log | head
for f in gpurun_out/probe_C*_ct*.log; do echo "== $f"; head -2 $f; grep "tail phase sweep\|L1 tail\|L2 tail" $f; done
