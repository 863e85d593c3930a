"""C2-shape predictor path loop timing: predict_props (+ append) then the
decode step on its props, vs each alone; CUDA events around 50-step loops."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_07719_b200.fluxattn import Engine, Predictor, SparseDecoder  # noqa: E402

eng = Engine(0)
dev = eng.device
B, HKV, G, D = 16, 8, 4, 128
dec = SparseDecoder(eng, B, HKV, G, D, 64, 131072 - 320, 256, max_new=1200, dtype="bf16")
dec.k.normal_()
dec.v.normal_()
dec.build_metadata()
q = torch.randn((B, 32, D), device=dev)
rs = np.random.default_rng(5)
params = {"w1": rs.standard_normal((256, 41)) * (2.0 / 41) ** 0.5, "b1": np.zeros(256),
          "w2": rs.standard_normal((384, 256)) * (2.0 / 256) ** 0.5, "b2": np.zeros(384),
          "w3": rs.standard_normal((3, 384)) * np.array([[1e-4], [2e-5], [1e-2]]),
          "b3": np.array([0.03, 0.005, 0.0]), "mu": np.zeros(41), "sigma": np.ones(41) * 50}
rec = dec.prefill_stats(q, tau=0.10, layer=0)
# as bench.py: normalization fitted on the first step's features, the
# streaming logit centred (about half the heads stream)
f0 = dec.decode_features(q, rec).reshape(-1, 41)
params["mu"] = f0.mean(0).cpu().numpy()
sd = f0.std(0)
params["sigma"] = torch.where(sd > 1e-9 * (1 + f0.mean(0).abs()), sd, torch.zeros_like(sd)).cpu().numpy()
pred = Predictor(eng, params)
z0 = torch.empty((B * 32, 3), dtype=torch.float64, device=dev)
pred(f0, z=z0)
params["b3"][2] = -float(z0[:, 2].median().item())
pred.close()
pred = Predictor(eng, params)
kn = torch.randn((B, HKV, D), device=dev)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)


def loop(fn, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


pp = dec.predict_props(q, rec, pred)
torch.cuda.synchronize()
print("streaming frac %.3f, retrieval groups %d" % (pp[2].float().mean().item(), 0))
print("props+append+step us %.1f" % loop(lambda: dec.step(q, props=dec.predict_props(q, rec, pred, append=(kn, kn)))))
print("props+step (no append) us %.1f" % loop(lambda: dec.step(q, props=dec.predict_props(q, rec, pred))))
print("props alone us %.1f" % loop(lambda: dec.predict_props(q, rec, pred)))
print("step alone us %.1f" % loop(lambda: dec.step(q, props=pp)))
print("step + append us %.1f" % loop(lambda: dec.step(q, props=pp, append=(kn, kn))))
base = dec.l_new
print("props+append alone us %.1f" % loop(lambda: dec.predict_props(q, rec, pred, append=(kn, kn))))


def grow_no_append():
    pp2 = dec.predict_props(q, rec, pred)
    dec.step(q, props=pp2)
    dec.l_new += 1


print("props+step, l_new grown by hand us %.1f" % loop(grow_no_append))


def fixed_len():
    dec.l_new = base
    dec.step(q, props=dec.predict_props(q, rec, pred, append=(kn, kn)))


print("props+append+step, l_new held us %.1f" % loop(fixed_len))
import time
t = time.time()
for _ in range(50):
    dec.step(q, props=dec.predict_props(q, rec, pred, append=(kn, kn)))
print("host time per props+append+step (no sync) us %.1f" % ((time.time() - t) / 50 * 1e6))
torch.cuda.synchronize()
print("l_new", dec.l_new)
# per-call host durations while l_new grows (a blocking call shows up here)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t = time.time()
    pp2 = dec.predict_props(q, rec, pred, append=(kn, kn))
    t1 = time.time()
    dec.step(q, props=pp2)
    t2 = time.time()
    ts.append(((t1 - t) * 1e6, (t2 - t1) * 1e6))
torch.cuda.synchronize()
print("host us per call (props, step):", " ".join("%.0f/%.0f" % x for x in ts))
