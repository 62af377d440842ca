# r02g: L2 capacity probe; level-1 sweep rate vs level-1 size
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/l2cap scripts/micro/l2_capacity.cu && timeout 120 /tmp/l2cap > gpurun_out/l2cap.log 2>&1
python -c "import paper_math_9809043_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
for n in 384 448 512; do
  timeout 300 python scripts/probe.py --config C5 --n $n --reps 2 > gpurun_out/probe_C5_n$n.log 2>&1
done
cat gpurun_out/l2cap.log
for n in 384 448 512; do grep -E "L1 halfsweep |solve " gpurun_out/probe_C5_n$n.log; done
