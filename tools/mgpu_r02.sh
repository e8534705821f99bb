#!/bin/bash
# Round-2 multi-GPU runs on one box (N = 2 and 4 when 4 GPUs are visible): PageRank bench
# lines, frontier workloads, parity vs the oracle, balance control run. Outputs gpurun_out/mg/.
set -u
O=gpurun_out/mg
mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29600
for n in 2 4; do
  [ $n -le $NG ] || continue
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p tools/mgpu_check.py --scale 18 > $O/check_s18_n$n.log 2>&1; echo "check n=$n rc=$?"
  p=$((p+1)); timeout 900 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --steps 20 --warmup 3 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo "bench n=$n rc=$?"
  for w in sssp-s26 cc-s24 lp-s22; do
    p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload $w --steps 20 --warmup 3 --no-e2e --no-parity > $O/wl_${w}_n$n.json 2> $O/wl_${w}_n$n.err; echo "wl $w n=$n rc=$?"
  done
done
p=$((p+1)); timeout 600 $TR --nproc-per-node 2 --master-port $p tools/balance_run.py --scale 20 > $O/balance_s20_n2.jsonl 2>&1; echo "balance rc=$?"
