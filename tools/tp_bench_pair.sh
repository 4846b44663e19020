#!/bin/bash
# NeMo-12B true-shape step at TP=1 and TP=2 (2-GPU box) -> profiles-style JSON lines
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python bench.py --model nemo12b --no-cpu --steps 20 > gpurun_out/nemo_tp1.json 2> gpurun_out/nemo_tp1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 \
    bench.py --model nemo12b --tp 2 --gpus 2 --no-cpu --steps 20 > gpurun_out/nemo_tp2.json 2> gpurun_out/nemo_tp2.err
