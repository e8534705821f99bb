#!/bin/bash
# Round-2 end-state multi-GPU records (run with gpurun --gpus 4): frontier workloads at N = 2 / 4
# after the line-aligned pack, LP at N = 1 / 2 / 4, and the S22 oracle check under torchrun.
set -u
O=gpurun_out/mg8
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=30210
for n in 2 4; do
  for w in sssp-s26 cc-s24 lp-s22; do
    st=12; [ $w = cc-s24 ] && st=8; [ $w = lp-s22 ] && st=15
    p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload $w --steps $st --warmup 3 --no-e2e --no-parity > $O/wl_${w}_n${n}.json 2> $O/wl_${w}_n${n}.err; echo "wl $w n=$n rc=$?"
  done
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p tools/mgpu_check.py --scale 22 > $O/check_s22_n$n.log 2>&1; echo "check n=$n rc=$?"
done
python bench.py --workload lp-s22 --steps 15 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-python-reference > $O/wl_lp-s22_n1.json 2> $O/wl_lp-s22_n1.err
