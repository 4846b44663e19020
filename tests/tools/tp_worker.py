"""One rank of a tensor-parallel engine group (used by tests/test_gpu_tp.py).
argv: rank size uid_hex golden_json_path -> prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2602_16760_b200 as sfg  # noqa: E402
import pyoracle as po  # noqa: E402

rank, size, uid = int(sys.argv[1]), int(sys.argv[2]), bytes.fromhex(sys.argv[3])
golden = json.load(open(sys.argv[4]))
cfg = po.tiny_cfg()
scfg = sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__})
eng = sfg.Engine(scfg, math=sfg.FAST, device=rank, tp=(size, rank, uid))
split = 1
srv = sfg.ServerEngine(eng, sfg.ServerConfig(split, cfg.n_layers - split))
la = sfg.LookaheadConfig(ngram_n=3, window_w=5, max_candidates_g=5)
out = []
for r in golden["runs"]:
    cl = sfg.SplitClient(eng, sfg.SplitConfig(split, split, sfg.F32 if r["wire_f32"] else sfg.F16), srv)
    res = (sfg.decode_sequential(cl, r["prompt"], r["max_new"]) if r["mode"] == 0
           else sfg.decode_lookahead(cl, r["prompt"], r["max_new"], la))
    out.append({"tokens": res.tokens, "step_accepted": res.step_accepted, "step_batch": res.step_batch})
print(json.dumps({"rank": rank, "runs": out}), flush=True)
