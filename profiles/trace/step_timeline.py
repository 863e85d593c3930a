"""One traced C2 step (drawn head properties): a single %globaltimer timeline
of the scorer, the selection (+ fused worklist) and the attention, relative to
the first scorer CTA's start (= k_prepare complete)."""
import os, sys, time, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["FLUXATTN_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfluxattn_b200.so")
from paper_2605_07719_b200 import _native as N
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder
eng = Engine(0); dev = eng.device
B, HKV, G, D = int(os.environ.get("TL_B", 16)), 8, 4, 128
ctx = 131072; l_cpu = ctx - 320
dec = SparseDecoder(eng, B, HKV, G, D, 64, l_cpu, 256, max_new=64, dtype="bf16")
dec.k.normal_(); dec.v.normal_(); dec.build_metadata()
rng = np.random.default_rng(1)
H = 32
props = tuple(torch.as_tensor(x, device=dev) for x in (rng.uniform(0.01, 0.05, (B, H)), rng.uniform(0, 0.01, (B, H)), (rng.random((B, H)) < 0.5).astype(np.int32)))
q = torch.randn((B, H, D), device=dev)
t = time.time()
while time.time() - t < 2.0:
    for i in range(50):
        dec.step(q, props=props)
    torch.cuda.synchronize()
for fn in ("fx_debug_sel_trace", "fx_debug_score_trace", "fx_debug_trace"):
    getattr(N.LIB, fn).argtypes = [C.c_void_p, C.c_int]
res = []
for rep in range(5):
    N.LIB.fx_debug_sel_trace_clear()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); dec.step(q, props=props); e1.record()
    torch.cuda.synchronize()
    sc = np.zeros(8 * 512, np.int64); N.LIB.fx_debug_score_trace(sc.ctypes.data, 8 * 148); sc = sc[:8 * 148].reshape(148, 8)
    nh = B * H
    se = np.zeros(16 * 8192, np.int64); N.LIB.fx_debug_sel_trace(se.ctypes.data, 16 * nh); se = se[:16 * nh].reshape(nh, 16)
    at = np.zeros(12 * 2048, np.int64); N.LIB.fx_debug_trace(at.ctypes.data, 12 * 148); at = at[:12 * 148].reshape(148, 12)
    t0 = sc[:, 0].min()
    us = lambda x: (x - t0) / 1e3
    live = se[:, 10] > 0
    wl = se[:, 9] > 0
    r = dict(step=e0.elapsed_time(e1) * 1e3,
             score_start_max=us(sc[:, 0].max()), score_first_box=np.median(us(sc[:, 2])),
             score_end_med=np.median(us(sc[:, 3])), score_end_max=us(sc[:, 3].max()),
             sel_start_min=us(se[live, 10].min()), sel_start_med=np.median(us(se[live, 10])), sel_start_max=us(se[live, 10].max()),
             sel_wait_done_med=np.median(us(se[se[:, 0] > 0, 0])),
             sel_head_end_med=np.median(us(se[live, 11])), sel_head_end_max=us(se[live, 11].max()),
             wl_end_max=us(se[wl, 9].max()),
             att_start_min=us(at[:, 0].min()), att_start_max=us(at[:, 0].max()),
             att_cons_end_med=np.median(us(at[:, 1])), att_cons_end_max=us(at[:, 1].max()),
             att_end_max=us(at[:, 8].max()))
    ph = se[se[:, 0] > 0][:, :6]
    for i in range(1, 6):
        r["sel_phase%d_mean" % i] = ((ph[:, i] - ph[:, i - 1]) / 1e3).mean()
        r["sel_phase%d_max" % i] = ((ph[:, i] - ph[:, i - 1]) / 1e3).max()
    res.append(r)
for k in res[0]:
    print("%-22s" % k, " ".join("%8.2f" % r[k] for r in res))
