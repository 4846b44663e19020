import sys, os, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2602_16760_b200 as sfg, pyoracle as po
cfg = po.desk_cfg(); port = po.Port(); m = port.model(cfg, bf16=True)
sc = sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__})
ep = sfg.Engine(sc, params=m.params()); es = sfg.Engine(sc)
rng = np.random.default_rng(0); h = rng.standard_normal((3, 64)).astype(np.float32)
a = ep.forward_layers(0, 8, h, [0,1,2], ep.bank(0, 8)); b = es.forward_layers(0, 8, h, [0,1,2], es.bank(0, 8))
print("seeded==params forward:", np.array_equal(a, b), np.abs(a-b).max())
print("embed eq", np.array_equal(ep.embed_at([1,2],[0,1]), es.embed_at([1,2],[0,1])))
prompt = [3,1,4,1,5,9,2,6]
toks, lg = m.generate(prompt, 3, want_logits=True)
for wire in (sfg.F32, sfg.F16):
    srv = sfg.ServerEngine(ep, sfg.ServerConfig(2, 6))
    cl = sfg.SplitClient(ep, sfg.SplitConfig(2, 2, wire), srv)
    first, row = cl.prefill(prompt, want_logits=True)
    print("wire", wire, "first", first, "port", toks[0], "row eq", np.array_equal(row, lg[0]), np.abs(row-lg[0]).max())
    l1 = cl.decode_step([first], [8], None, [], None)
    print("  step1 argmax", int(np.argmax(l1[0])), "port", toks[1], "eq", np.array_equal(l1[0], lg[1]), np.abs(l1[0]-lg[1]).max())
    for frames in (True,):
        cl = sfg.SplitClient(ep, sfg.SplitConfig(2, 2, wire), srv, frames=True)
        first, row = cl.prefill(prompt, want_logits=True)
        print("  frames first", first, "row eq", np.array_equal(row, lg[0]), np.abs(row-lg[0]).max())
import ctypes as C
from paper_2602_16760_b200 import _lib
x = (rng.standard_normal(100000) * 10).astype(np.float32)
x[:6] = [1e6, -70000, 65519, 1e-8, 3e-8, -0.0]
y = np.empty_like(x); cc = C.c_uint64()
_lib.check(_lib.lib().sfg_selftest_wire_roundtrip(x.ctypes.data_as(C.POINTER(C.c_float)), y.ctypes.data_as(C.POINTER(C.c_float)), len(x), C.byref(cc)))
exp = np.array([port.f16_to_f32(port.f32_to_f16(float(v))) for v in x], dtype=np.float32)
print("roundtrip eq", np.array_equal(y.view(np.uint32), exp.view(np.uint32)), "clamped", cc.value)
# linked vs frames f16 step logits
srv = sfg.ServerEngine(ep, sfg.ServerConfig(2, 6))
res = []
for frames in (False, True):
    cl = sfg.SplitClient(ep, sfg.SplitConfig(2, 2, sfg.F16), srv, session_id="s%d" % frames, frames=frames)
    first, row = cl.prefill(prompt, want_logits=True)
    res.append((first, row))
print("linked vs frames prefill", res[0][0], res[1][0], np.abs(res[0][1]-res[1][1]).max())
