#!/bin/bash
# torchrun path of bench.py (N=1 under torchrun) and the reference arm with many steps
set -x
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_torchrun.log 2>&1; echo "torchrun rc=$?"
tail -1 gpurun_out/r02_bench_torchrun.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r02_bench_ref10.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r02_bench_ref10.log | cut -c1-400
