"""Phase times of the clustered decode-features kernel (k_feat_fused) at C2,
and the fx_predict_props total (features + the tiled predictor layers)."""
import os, sys, time, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["FLUXATTN_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfluxattn_b200.so")
from paper_2605_07719_b200 import _native as N
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder, Predictor
eng = Engine(0); dev = eng.device
B, HKV, G, D = 16, 8, 4, 128
ctx = 131072; l_cpu = ctx - 320
dec = SparseDecoder(eng, B, HKV, G, D, 64, l_cpu, 256, max_new=300, dtype="bf16")
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.time()
while time.time() - t < 2.0:
    for i in range(50):
        dec.predict_props(q, rec, pred)
    torch.cuda.synchronize()
e0.record()
for i in range(100):
    dec.predict_props(q, rec, pred)
e1.record(); torch.cuda.synchronize()
print("predict_props us %.2f (l_new %d)" % (e0.elapsed_time(e1) / 100 * 1e3, dec.l_new))
tr = np.zeros(16 * 1024, np.int64)
N.LIB.fx_debug_fp_trace.argtypes = [C.c_void_p, C.c_int]
N.LIB.fx_debug_fp_trace(tr.ctypes.data, 16 * 128)
t = tr[:16 * 128].reshape(128, 16)
t0 = t[:, 0].min()
names = ["start", "q staged", "sink", "local", "new", "features", "feats out", "L0 begin", "L0 data", "L0 scores", "L0 weights", "L0 o"]
N.LIB.fx_ctx_set_timing(eng.ctx, 1)
for i in range(20):
    dec.predict_props(q, rec, pred)
N.LIB.fx_ctx_set_timing(eng.ctx, 0)
for i, nm in enumerate(names):
    x = (t[:, i] - t0) / 1e3
    print("%-12s min %7.2f median %7.2f max %7.2f" % (nm, x.min(), np.median(x), x.max()))

cyc = (t[:, 15] - t[:, 14]).astype(np.float64)
ns = (t[:, 6] - t[:, 0]).astype(np.float64)
print("effective SM clock over the kernel: median %.0f MHz" % np.median(cyc / ns * 1e3))
