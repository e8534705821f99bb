export GXB_TILE_MINBLOCKS=6
python tools/probe.py --scale 26 --iters 3 > gpurun_out/probe26c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_tile -s 1 -c 1 -o gpurun_out/prof_tile26c python tools/probe.py --scale 26 --iters 3 > gpurun_out/ncu_tile26c.log 2>&1
tail -2 gpurun_out/ncu_tile26c.log
