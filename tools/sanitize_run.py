"""Workload for compute-sanitizer (memcheck / racecheck / synccheck) on the
tiny config: exercises every kernel family of the product path once.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py

* FAST lookahead decode through the device-linked client: the layer-stack
  megakernel (per-row attention), LM head + argmax partials, verify tail,
  in-place KV compaction driven by the step meta (kv_compact_meta_kernel),
  wire pack/unpack, CUDA-graph replay;
* the frame-level server with two sessions batched in one weight pass
  (handle_batch: cross-session rowinfo in the megakernel);
* a prompt pass > 16 rows (per-GEMM path: gemm_kernel<EPI, 5>, prep, attention_fast);
* seam-2 resolve with a keep list longer than one compaction chunk
  (kv_compact_kernel, 64-row chunks);
* the EXACT path decode (serial CUDA-core kernels).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_16760_b200 as sfg  # noqa: E402
import pyoracle as po  # noqa: E402
import wirepy  # noqa: E402


def main():
    cfg = po.tiny_cfg()
    port = po.Port()
    m = port.model(cfg, bf16=True)
    mc = sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__})
    la = sfg.LookaheadConfig(ngram_n=3, window_w=5, max_candidates_g=5)
    prompt = [7, 7, 7, 7, 7, 7, 7, 7]
    feng = sfg.Engine(mc, math=sfg.FAST, params=m.params())
    srv = sfg.ServerEngine(feng, sfg.ServerConfig(1, cfg.n_layers - 1))
    out = sfg.decode_lookahead(sfg.SplitClient(feng, sfg.SplitConfig(1, 1, sfg.F16), srv), prompt, 12, la)
    print("FAST linked decode:", out.tokens)
    # frame-level server, two sessions' steps in one weight pass
    rng = np.random.default_rng(0)
    H = cfg.hidden_dim
    for sid in ("a", "b"):
        srv.handle(wirepy.hidden_request("prompt", sid, rng.standard_normal((4, H)).astype(np.float32), list(range(4))))
    frames = [wirepy.hidden_request("step", sid, rng.standard_normal((3, H)).astype(np.float32), [4, 5, 6])
              for sid in ("a", "b")]
    resp = srv.handle_batch(frames)
    print("batched:", [wirepy.decode(r)[0]["kind"] for r in resp], "shared passes", srv.shared_passes())
    # prompt pass > 16 rows and a long keep list (chunked compaction)
    b = feng.bank(1, cfg.n_layers - 1)
    h = rng.standard_normal((100, H)).astype(np.float32)
    feng.forward_layers(1, cfg.n_layers - 1, h, list(range(100)), b)
    b.mark_committed(0)
    b.resolve(list(range(1, 91)))  # 90 kept rows, shifted by one: not the identity
    print("bank after resolve:", b.len(), b.committed_len())
    # EXACT path
    eeng = sfg.Engine(mc, math=sfg.EXACT, params=m.params())
    esrv = sfg.ServerEngine(eeng, sfg.ServerConfig(1, cfg.n_layers - 1))
    out = sfg.decode_lookahead(sfg.SplitClient(eeng, sfg.SplitConfig(1, 1, sfg.F16), esrv), prompt, 8, la)
    print("EXACT decode:", out.tokens)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
