"""Phase times (%globaltimer) of the decode-feature kernels at C2 (16 x 8
groups, 128K, bf16): k_feat_part per CTA (start, item ends, end) and
k_feat_final per CTA (start, before / after the grid-dependency wait, heads
merged, cluster exchange done, layer 1 done), one fx_predict_props call."""
import os, sys, time, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["FLUXATTN_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfluxattn_b200.so")
from paper_2605_07719_b200 import _native as N
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder, Predictor
eng = Engine(0); dev = eng.device
B, HKV, G, D = 16, 8, 4, 128
ctx = 131072; l_cpu = ctx - 320
dec = SparseDecoder(eng, B, HKV, G, D, 64, l_cpu, 256, max_new=640, dtype="bf16")
dec.k.normal_(); dec.v.normal_(); dec.build_metadata()
q = torch.randn((B, 32, D), device=dev)
rs = np.random.default_rng(5)
params = {"w1": rs.standard_normal((256, 41)) * (2.0 / 41) ** 0.5, "b1": np.zeros(256),
          "w2": rs.standard_normal((384, 256)) * (2.0 / 256) ** 0.5, "b2": np.zeros(384),
          "w3": rs.standard_normal((3, 384)) * 1e-2, "b3": np.array([0.03, 0.005, 0.0]),
          "mu": np.zeros(41), "sigma": np.ones(41) * 50}
pred = Predictor(eng, params)
rec = dec.prefill_stats(q, tau=0.10, layer=0)
dec.l_new = int(sys.argv[1]) if len(sys.argv) > 1 else 100
t = time.time()
while time.time() - t < 1.0:
    for i in range(50):
        dec.predict_props(q, rec, pred)
    torch.cuda.synchronize()
N.LIB.fx_debug_fp_trace.argtypes = [C.c_void_p, C.c_int]
for rep in range(3):
    torch.cuda.synchronize()
    dec.predict_props(q, rec, pred)
    torch.cuda.synchronize()
    tr = np.zeros(16 * 2048, np.int64)
    N.LIB.fx_debug_fp_trace(tr.ctypes.data, 16 * 2048)
    t = tr.reshape(2048, 16)
    part = t[:296]
    part = part[part[:, 0] > 0]
    fin = t[1024:1024 + 128]
    t0 = part[:, 0].min()
    us = lambda x: (x - t0) / 1e3
    print("rep", rep, "l_new", dec.l_new)
    print("  part: start min %.2f max %.2f | item0 end med %.2f | end med %.2f max %.2f" % (
        us(part[:, 0].min()), us(part[:, 0].max()), np.median(us(part[:, 2])), np.median(us(part[:, 1])), us(part[:, 1].max())))
    for i, nm in [(12, "it1 top"), (13, "it1 data"), (9, "it1 scores"), (10, "it1 exp"), (11, "it1 PV"), (3, "it1 end")]:
        x = us(part[:, i])
        print("  part %-9s min %7.2f med %7.2f max %7.2f" % (nm, x.min(), np.median(x), x.max()))
    for i, nm in [(0, "start"), (1, "pre-wait"), (2, "post-wait"), (6, "m/z in"), (7, "weights"), (8, "outputs"), (9, "norms"), (3, "heads"), (4, "cluster"), (5, "layer1")]:
        x = us(fin[:, i])
        print("  final %-9s min %7.2f med %7.2f max %7.2f" % (nm, x.min(), np.median(x), x.max()))
    cyc = (fin[:, 15] - fin[:, 14]).astype(np.float64)
    ns = (fin[:, 5] - fin[:, 0]).astype(np.float64)
    print("  effective SM clock over k_feat_final: median %.0f MHz" % np.median(cyc / ns * 1e3))
