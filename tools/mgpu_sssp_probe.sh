#!/bin/bash
# SSSP S26 multi-GPU breakdown: per-round step times (bench) and per-phase times (mgpu_rounds)
set -u
O=gpurun_out/mg3
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29800
for n in 2 4; do
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload sssp-s26 --steps 12 --warmup 3 --no-e2e --no-parity > $O/wl_sssp_n$n.json 2> $O/wl_sssp_n$n.err; echo "wl n=$n rc=$?"
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p tools/mgpu_rounds.py sssp 26 > $O/rounds_sssp_n$n.log 2>&1; echo "rounds n=$n rc=$?"
done
python bench.py --workload sssp-s26 --steps 12 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-python-reference > $O/wl_sssp_n1.json 2> $O/wl_sssp_n1.err
