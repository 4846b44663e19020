cd ${GRAFT_REPO_ROOT:-.}
# NeMo-12B step under SFG_MEGA_ALIGN settings at TP=2 and TP=1 (2-GPU box)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['server_ms_per_step'],4))"; }
port=29600
for al in 85 70 50 0; do
  port=$((port+1))
  echo "== tp2 ALIGN=$al"; SFG_MEGA_ALIGN=$al timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --model nemo12b --tp 2 --gpus 2 --no-sweep --no-cpu --steps 10 2>/dev/null | p
  echo "== tp1 ALIGN=$al"; SFG_MEGA_ALIGN=$al timeout 300 python bench.py --model nemo12b --no-sweep --no-cpu --steps 10 2>/dev/null | p
done
