run() { echo "== $*"; env "$@" timeout 300 python bench.py --no-sweep --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['server_ms_per_step'],4))"; }
run SFG_MEGA_BPF=0
run SFG_MEGA_BPF=8 SFG_MEGA_BPF_CYC=1000
run SFG_MEGA_BPF=16 SFG_MEGA_BPF_CYC=1000
run SFG_MEGA_BPF=32 SFG_MEGA_BPF_CYC=2000
run SFG_MEGA_BPF=16 SFG_MEGA_BPF_CYC=400
run SFG_MEGA_PF=8
run SFG_MEGA_ALIGN=0
run SFG_MEGA_ALIGN=60
