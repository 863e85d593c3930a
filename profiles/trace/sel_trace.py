import os, sys, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["FLUXATTN_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfluxattn_b200.so")
from paper_2605_07719_b200 import _native as N
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder
eng = Engine(0); dev = eng.device
# shape from the environment (default C2; C3: SEL_B=8 SEL_HKV=4 SEL_G=7 SEL_CTX=262144)
B, HKV, G, D = int(os.environ.get("SEL_B", 16)), int(os.environ.get("SEL_HKV", 8)), int(os.environ.get("SEL_G", 4)), 128
ctx = int(os.environ.get("SEL_CTX", 131072)); l_cpu = ctx - 320
dec = SparseDecoder(eng, B, HKV, G, D, 64, l_cpu, 256, max_new=64, dtype="bf16")
dec.k.normal_(); dec.v.normal_(); dec.build_metadata()
rng = np.random.default_rng(1)
H = HKV * G
props = tuple(torch.as_tensor(x, device=dev) for x in (rng.uniform(0.01, 0.05, (B, H)), rng.uniform(0, 0.01, (B, H)), (rng.random((B, H)) < 0.5).astype(np.int32)))
q = torch.randn((B, H, D), device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(5):
    ev[0].record(); dec.step(q, props=props); ev[1].record()
torch.cuda.synchronize()
N.LIB.fx_debug_sel_trace_clear()
torch.cuda.synchronize()
dec.step(q, props=props)
torch.cuda.synchronize()
print("step ms %.3f" % ev[0].elapsed_time(ev[1]))
tr = np.zeros(16 * 8192, np.int64)
N.LIB.fx_debug_sel_trace.argtypes = [C.c_void_p, C.c_int]
N.LIB.fx_debug_sel_trace(tr.ctypes.data, 16 * B * H)
t = tr[:16 * B * H].reshape(B * H, 16)
t0 = t[:, 10].min()
print("kernel CTA start spread (us): %.2f" % ((t[:, 10].max() - t0) / 1e3))
print("select_head end (us): median %.2f max %.2f" % (np.median(t[:, 11] - t0) / 1e3, (t[:, 11].max() - t0) / 1e3))
wl = t[:, 8] > 0
print("worklist CTAs", wl.sum(), "start max %.2f  end max %.2f  dur mean %.2f max %.2f" % ((t[wl, 8].max() - t0) / 1e3, (t[wl, 9].max() - t0) / 1e3, (t[wl, 9] - t[wl, 8]).mean() / 1e3, (t[wl, 9] - t[wl, 8]).max() / 1e3))
live = t[:, 0] > 0
ph = t[live][:, :6] - t0
for i in range(1, 6):
    d = (ph[:, i] - ph[:, i - 1]) / 1e3
    print("phase %d: mean %.2f us  max %.2f" % (i, d.mean(), d.max()))

w = t[wl]
for a, b, name in [(8, 12, "stage"), (12, 13, "count+scan"), (13, 14, "emit"), (14, 9, "tail")]:
    ok = (w[:, a] > 0) & (w[:, b] > 0)
    d = (w[ok, b] - w[ok, a]) / 1e3
    print("worklist %s: mean %.2f max %.2f (n=%d)" % (name, d.mean(), d.max(), ok.sum()))
print("worklist start after select_head end of same CTA: mean %.2f" % (((w[:, 8] - w[:, 11]) / 1e3).mean()))
lv = t[:, 11] > 0
nc = t[:, 6] & 0xffffffff; nd = t[:, 6] >> 32; kk = t[:, 7] & 0xffffffff; nb = t[:, 7] >> 32
end = (t[:, 11] - t0) / 1e3
for blk_n in sorted(set(nb[lv].tolist())):
    m = lv & (nb == blk_n)
    print("nblk %5d heads %3d end median %.2f max %.2f  cand median %d max %d  k median %d" % (blk_n, m.sum(), np.median(end[m]), end[m].max(), np.median(nc[m]), nc[m].max(), np.median(kk[m])))
live = t[:, 0] > 0
for i in range(1, 6):
    d = (t[:, i] - t[:, i - 1]) / 1e3
    print("phase %d by nblk:" % i, ", ".join("%d: %.2f" % (b, d[live & (nb == b)].mean()) for b in sorted(set(nb[live].tolist()))))
