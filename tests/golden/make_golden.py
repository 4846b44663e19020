"""Regenerates tests/golden/*.json from the UNMODIFIED reference compiled in
place (oracle/_ref/libsplitf_ref.so, built by `make -C oracle ref` from
/root/reference/proj/src).  Run here (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin both the C restatement (oracle/liboracle.so) and the B200
engine to the reference's own outputs on the GPU box, where /root/reference
is absent.  Logits are stored as SHA-256 digests of their fp32 bytes.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402


def digest(a):
    return hashlib.sha256(a.tobytes()).hexdigest()


def decode_cases(ref, cfg, split, prompts, max_new, name):
    m = ref.model(cfg, bf16=True)
    runs = []
    for wire_f32 in (1, 0):
        for mode in (0, 2):
            for pi, prompt in enumerate(prompts):
                dc = po.DecodeCfg(mode=mode, prefix_layers=split, suffix_layers=split, wire_f32=wire_f32,
                                  window_w=5, ngram_n=3, max_candidates_g=5)
                r = ref.decode(m, dc, prompt, max_new, want_logits=True)
                runs.append({"mode": mode, "wire_f32": wire_f32, "prompt": list(map(int, prompt)),
                             "max_new": max_new, "tokens": r.tokens, "step_batch": r.step_batch,
                             "step_accepted": r.step_accepted, "logits_sha256": digest(r.logits)})
    cfgd = {k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}
    return {"name": name, "source": "oracle/_ref (reference decode_* via SimPipeline pieces, ref_shim.cpp)",
            "config": cfgd, "weights": "init_weights(seed) rounded to bf16 RNE", "split": split,
            "lookahead": {"W": 5, "N": 3, "G": 5}, "runs": runs}


def main():
    ref = po.Ref()
    # tiny = BASELINE config 1 (4 layers, d=256, GQA 4q/2kv x 64, 1+1 split)
    tiny = po.tiny_cfg()
    rep = ref.corpus("repetitive", tiny.vocab_size, 4, 24, 100)
    rnd = ref.corpus("random", tiny.vocab_size, 4, 24, 101)
    out = decode_cases(ref, tiny, 1, rep[:2] + rnd[:2], 32, "tiny")
    with open(os.path.join(HERE, "ref_decode_tiny.json"), "w") as f:
        json.dump(out, f, indent=1)
    # desk = reference default ModelConfig, 2+2 split
    desk = po.desk_cfg()
    rep = ref.corpus("repetitive", desk.vocab_size, 3, 12, 100)
    rnd = ref.corpus("random", desk.vocab_size, 3, 12, 101)
    out = decode_cases(ref, desk, 2, rep + rnd, 40, "desk")
    with open(os.path.join(HERE, "ref_decode_desk.json"), "w") as f:
        json.dump(out, f, indent=1)
    # monolithic traces (fp32 and bf16 weights)
    mono = []
    for bf16 in (False, True):
        m = ref.model(desk, bf16=bf16)
        for prompt in ([3, 1, 4, 1, 5, 9, 2, 6], [1, 2, 3, 4], [7]):
            toks, lg = m.generate(prompt, 24, want_logits=True)
            mono.append({"bf16": bf16, "prompt": prompt, "tokens": toks, "logits_sha256": digest(lg)})
    with open(os.path.join(HERE, "ref_monolithic_desk.json"), "w") as f:
        json.dump({"source": "oracle/_ref generate_monolithic_traced", "runs": mono}, f, indent=1)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
