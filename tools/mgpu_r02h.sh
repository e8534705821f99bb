#!/bin/bash
# CC S24 at N = 1 / 2 / 4 after push_alpha 10 (run with gpurun --gpus 4)
set -u
O=gpurun_out/mg9
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=30410
python bench.py --workload cc-s24 --steps 8 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-python-reference > $O/wl_cc-s24_n1.json 2> $O/wl_cc-s24_n1.err
for n in 2 4; do
  p=$((p+1)); timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --workload cc-s24 --steps 8 --warmup 3 --no-e2e --no-parity > $O/wl_cc-s24_n$n.json 2> $O/wl_cc-s24_n$n.err; echo "cc n=$n rc=$?"
done
for n in 1 2 4; do echo "n=$n $(grep -o '"value": [0-9.]*' $O/wl_cc-s24_n$n.json | head -1)"; done
