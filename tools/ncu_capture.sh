#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root, ONE GPU):
#   1. the bench command itself must have exited 0 without ncu first;
#   2. launch list of the same command (per-launch durations, cold/serialised);
#   3. one --set full capture of the dominant kernel (the layer-stack megakernel).
set -e
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 3 --no-sweep --no-cpu"
timeout 600 python bench.py $ARGS > gpurun_out/ncu_pre_bench.txt
# decode-step kernels only (the weight-init conversion/relayout kernels are excluded)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:'mega_kernel|head_argmax|argmax|verify|pack|unpack|embed|kv_compact|link_delay|attention|gemm|rmsnorm' \
    --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mega_kernel --launch-skip 4 -c 1 \
    -o gpurun_out/mega_full -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/mega_full.ncu-rep --page raw --csv > gpurun_out/mega_full_raw.csv
ncu -i gpurun_out/mega_full.ncu-rep --page details --csv > gpurun_out/mega_full_details.csv
