"""Per-CTA phase times of the generic (f32) attention kernel at the C1 shape
(batch 1, 8 groups, 32K, f32, fixed (64, 0.05)): start, after the grid wait,
after the run starts, first box staged, end."""
import os, sys, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["FLUXATTN_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfluxattn_b200.so")
from paper_2605_07719_b200 import _native as N
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder
eng = Engine(0); dev = eng.device
dec = SparseDecoder(eng, 1, 8, 4, 128, 64, 32768 - 320, 256, max_new=64, dtype="f32")
dec.k.normal_(); dec.v.normal_(); dec.build_metadata()
q = torch.randn((1, 32, 128), device=dev)
for i in range(20):
    dec.step(q, fixed=(64, 0.05))
torch.cuda.synchronize()
N.LIB.fx_debug_gtrace.argtypes = [C.c_void_p, C.c_int]
tr = np.zeros(8 * 2048, np.int64)
N.LIB.fx_debug_gtrace(tr.ctypes.data, 8 * 2048)
t = tr.reshape(2048, 8)
live = t[:, 0] > 0
t = t[live]
t0 = t[:, 0].min()
us = lambda x: (x - t0) / 1e3
print("CTAs", live.sum())
for i, nm in [(0, "start"), (1, "after wait"), (2, "run starts"), (3, "first box staged"), (5, "end")]:
    x = us(t[t[:, i] > 0, i])
    print("%-18s min %7.2f med %7.2f max %7.2f" % (nm, x.min(), np.median(x), x.max()))
