"""fx_predict_props at the C2 shape (16 x 8 groups, 128K, 100 decoded rows):
the feature kernels (partials + clustered merge with layer 1) + layers 2 + 3, for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_07719_b200.fluxattn import Engine, Predictor, SparseDecoder  # noqa: E402

eng = Engine(0)
dev = eng.device
B, HKV, G, D = 16, 8, 4, 128
dec = SparseDecoder(eng, B, HKV, G, D, 64, 131072 - 320, 256, max_new=128, dtype="bf16")
dec.k.normal_()
dec.v.normal_()
dec.build_metadata()
q = torch.randn((B, 32, D), device=dev)
rs = np.random.default_rng(5)
params = {"w1": rs.standard_normal((256, 41)) * (2.0 / 41) ** 0.5, "b1": np.zeros(256),
          "w2": rs.standard_normal((384, 256)) * (2.0 / 256) ** 0.5, "b2": np.zeros(384),
          "w3": rs.standard_normal((3, 384)) * 1e-2, "b3": np.array([0.03, 0.005, 0.0]),
          "mu": np.zeros(41), "sigma": np.ones(41) * 50}
pred = Predictor(eng, params)
rec = dec.prefill_stats(q, tau=0.10, layer=0)
dec.l_new = 100
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    dec.predict_props(q, rec, pred)
torch.cuda.synchronize()
print("ok")
