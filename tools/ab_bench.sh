#!/bin/bash
# A/B the decode step over library builds / env settings (dev tool):
#   tools/ab_bench.sh "label|ENV=.. ENV2=.." ...   (LIB=ablib/x.so swaps that build in place)
mkdir -p gpurun_out
SO=paper_2602_16760_b200/libsfg.so
cp $SO /tmp/libsfg_orig.so
for spec in "$@"; do
  label=${spec%%|*}; envs=${spec#*|}
  lib=$(echo "$envs" | tr ' ' '\n' | sed -n 's/^LIB=//p')
  if [ -n "$lib" ]; then cp "$lib" $SO; else cp /tmp/libsfg_orig.so $SO; fi
  envs=$(echo "$envs" | tr ' ' '\n' | grep -v '^LIB=' | tr '\n' ' ')
  env $envs timeout 600 python bench.py --no-sweep --no-cpu --steps 10 $BENCH_ARGS > gpurun_out/ab_$label.txt 2> gpurun_out/ab_$label.err
  python - "$label" <<'PY'
import json, sys
label = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{label}.txt").read().strip().splitlines()[-1])
    ks = d["kernel_classes"].get("layer_stack", {})
    print(f"{label:14s} ms/step {d['ms_per_step']:.3f}  layer_stack ms {ks.get('ms', 0) / d['steps']:.3f}/step"
          f"  achieved {d['roofline']['achieved']:.0f} GB/s  e2e {d['e2e']['ms_per_step']:.3f} ms")
except Exception as e:
    print(label, "FAILED", e, open(f"gpurun_out/ab_{label}.err").read()[-500:])
PY
done
cp /tmp/libsfg_orig.so $SO
