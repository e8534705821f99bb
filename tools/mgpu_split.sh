#!/bin/bash
# Split rounds A/B at N = 4 (gpurun --gpus 4): SSSP S26 / CC S24 with the local-source pass
# beside the exchange (GXB_SPLIT_OVERLAP=1, reserve 0 / 16 / 32 SMs) against whole rounds.
set -u
O=gpurun_out/split
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
p=30310
for rep in 1 2; do
for cfg in "0 16" "1 0" "1 16" "1 32"; do
  set -- $cfg
  for w in sssp-s26 cc-s24; do
    st=12; [ $w = cc-s24 ] && st=8
    p=$((p+1)); GXB_SPLIT_OVERLAP=$1 GXB_SPLIT_RESERVE_SMS=$2 timeout 600 $TR --master-port $p bench.py --gpus 4 --workload $w --steps $st --warmup 3 --no-e2e --no-parity > $O/wl_${w}_s$1_r$2_$rep.json 2> $O/wl_${w}_s$1_r$2_$rep.err
    echo "$w split=$1 reserve=$2 rep=$rep rc=$? $(grep -o '"value": [0-9.]*' $O/wl_${w}_s$1_r$2_$rep.json | head -1)"
  done
done
done
