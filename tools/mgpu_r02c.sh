#!/bin/bash
# dense mirror exchange vs per-peer records for the frontier workloads at N = 2 / 4
set -u
O=gpurun_out/mg4
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29950
for n in 2 4; do
  for w in sssp-s26 cc-s24 lp-s22; do
    st=12; [ $w = cc-s24 ] && st=8; [ $w = lp-s22 ] && st=15
    for df in 0.25 0; do
      p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload $w --steps $st --warmup 3 --no-e2e --no-parity --dense-frac $df > $O/wl_${w}_n${n}_df$df.json 2> $O/wl_${w}_n${n}_df$df.err; echo "wl $w n=$n df=$df rc=$?"
    done
  done
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p tools/mgpu_check.py --scale 22 > $O/check_s22_n$n.log 2>&1; echo "check n=$n rc=$?"
done
