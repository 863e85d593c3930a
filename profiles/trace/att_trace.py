import os, sys, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["FLUXATTN_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfluxattn_b200.so")
from paper_2605_07719_b200 import _native as N
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder
eng = Engine(0); dev = eng.device
B, HKV, G, D = 16, 8, 4, 128
ctx = 131072; l_cpu = ctx - 320
dec = SparseDecoder(eng, B, HKV, G, D, 64, l_cpu, 256, max_new=64, dtype="bf16")
dec.k.normal_(); dec.v.normal_(); dec.build_metadata()
rng = np.random.default_rng(1)
H = 32
props = tuple(torch.as_tensor(x, device=dev) for x in (rng.uniform(0.01, 0.05, (B, H)), rng.uniform(0, 0.01, (B, H)), (rng.random((B, H)) < 0.5).astype(np.int32)))
q = torch.randn((B, H, D), device=dev)
for i in range(6):
    dec.step(q, props=props)
torch.cuda.synchronize()
tr = np.zeros(12 * 2048, np.int64)
N.LIB.fx_debug_trace.argtypes = [C.c_void_p, C.c_int]
N.LIB.fx_debug_trace(tr.ctypes.data, 12 * 148)
t = tr[:12 * 148].reshape(148, 12)
t0 = t[:, 0].min()
st = (t[:, 0] - t0) / 1e3; ce = (t[:, 1] - t0) / 1e3; fe = (t[:, 8] - t0) / 1e3
print("CTA start: min %.2f max %.2f us" % (st.min(), st.max()))
print("consumer end: min %.2f median %.2f max %.2f" % (ce.min(), np.median(ce), ce.max()))
print("finish end: min %.2f median %.2f max %.2f" % (fe.min(), np.median(fe), fe.max()))
print("runs/CTA mean %.1f, tiles/CTA mean %.1f min %d max %d" % (t[:, 2].mean(), t[:, 3].mean(), t[:, 3].min(), t[:, 3].max()))
print("consumer wait (us) mean %.2f, first %.2f, flush %.2f; producer wait %.2f" % (t[:, 4].mean() / 1e3, t[:, 5].mean() / 1e3, t[:, 6].mean() / 1e3, t[:, 7].mean() / 1e3))
print("finish merges: nruns mean %.2f, merged-by-me mean %.2f" % (t[:, 9].mean(), t[:, 10].mean()))
print("finish duration mean %.2f max %.2f" % ((fe - ce).mean(), (fe - ce).max()))
sm = t[:, 11]
order = np.argsort(ce)
print("slowest 10 CTAs: id", order[-10:], "sm", sm[order[-10:]], "tiles", t[order[-10:], 3], "runs", t[order[-10:], 2])
print("fastest 10 CTAs: id", order[:10], "sm", sm[order[:10]], "tiles", t[order[:10], 3], "runs", t[order[:10], 2])
print("corr(end, sm) %.3f corr(end, cta) %.3f corr(end, tiles) %.3f corr(end, runs) %.3f" % (
    np.corrcoef(ce, sm)[0, 1], np.corrcoef(ce, np.arange(148))[0, 1], np.corrcoef(ce, t[:, 3])[0, 1], np.corrcoef(ce, t[:, 2])[0, 1]))
lo = sm < 74
print("mean end: sm<74 %.2f  sm>=74 %.2f" % (ce[lo].mean(), ce[~lo].mean()))
print("mean end: even sm %.2f odd sm %.2f" % (ce[sm % 2 == 0].mean(), ce[sm % 2 == 1].mean()))
