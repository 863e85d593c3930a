"""Generate the golden vectors in tests/golden/ from the COMPILED REFERENCE
(oracle/_ref/libfluxref.so, built from /root/reference/proj/src by
oracle/Makefile).  Run here (where /root/reference exists):

    python tests/golden/make_golden.py

Each fixture stores the inputs (reference-generated synthetic workload,
workload.cpp:154-308) and the reference's outputs of the hot-path functions.
The files are small; the GPU box never needs /root/reference to use them.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import RefOracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    ref = RefOracle()
    spec = dict(heads=8, group_size=4, head_dim=64, context_len=1024, layers=1, decode_steps=2,
                seed=11, sink_frac=0.25, streaming_frac=0.25, retrieval_frac=0.5)
    w = ref.generate(**spec)
    l_sink, l_local = 64, 256
    l_cpu = 1024 - l_sink - l_local
    out = {"spec": json.dumps(spec)}
    for g in range(2):
        k, v = w.group_kv(0, g)
        nk, nv = w.new_kv(0, 0)
        out[f"k{g}"] = np.vstack([k, nk[g:g + 1]])
        out[f"v{g}"] = np.vstack([v, nv[g:g + 1]])
    out["q"] = w.queries(0, 1)
    out["archetypes"] = np.array([w.archetype(0, h) for h in range(8)], np.int32)
    # metadata at every candidate granularity (group 0)
    kc = out["k0"][l_sink:l_sink + l_cpu]
    for blk in (1, 16, 32, 64, 128):
        mins, maxs = ref.build_metadata(kc, blk)
        out[f"mins_{blk}"], out[f"maxs_{blk}"] = mins, maxs
    # scores and top-k for the 4 heads of group 0
    for blk in (16, 64):
        mins, maxs = out[f"mins_{blk}"], out[f"maxs_{blk}"]
        nblk = len(mins)
        out[f"scores_{blk}"] = np.array([[ref.block_score(out["q"][h], mins, maxs, blk, l_cpu, b)
                                          for b in range(nblk)] for h in range(4)])
        for kk in (1, 3, 9, nblk + 2):
            sels = [ref.topk_blocks(out["q"][h], mins, maxs, blk, l_cpu, kk) for h in range(4)]
            out[f"topk_{blk}_{kk}"] = np.array([np.pad(s["blocks"].astype(np.int64), (0, nblk + 2 - len(s["blocks"])),
                                                       constant_values=-1) for s in sels])
    # execute_task for both groups at a given plan
    budgets = np.array([0.05, 0.0, 0.2, 1.0])
    for g in range(2):
        out[f"exec_{g}"] = ref.execute_group(out[f"k{g}"], out[f"v{g}"], (l_sink, l_cpu, l_local, 1),
                                             out["q"][g * 4:(g + 1) * 4], 32, budgets)
    # selector on drawn head properties
    rng = np.random.default_rng(3)
    props = np.stack([rng.uniform(-0.05, 0.2, (64, 4)), rng.uniform(-0.01, 0.03, (64, 4)),
                      (rng.random((64, 4)) < 0.4)], axis=-1)
    out["props"] = props
    plans = [ref.plan_group(p[:, 0], p[:, 1], p[:, 2].astype(np.int32), 130752) for p in props]
    out["plan_blk"] = np.array([p["block_size"] for p in plans], np.int32)
    out["plan_vol"] = np.array([p["volume"] for p in plans])
    out["plan_cand"] = np.array([p["candidate_volumes"] for p in plans])
    out["plan_bud"] = np.array([p["budgets"] if len(p["budgets"]) else np.zeros(4) for p in plans])
    # predictor: make_model(5) with nontrivial norms (parameters are regenerated
    # from the seed by the oracle's make_model restatement)
    m = ref.make_model(5)
    mu = rng.standard_normal(41)
    sigma = np.abs(rng.standard_normal(41)) + 0.2
    sigma[7] = 0.0
    m.set_norms(mu, sigma)
    feats = rng.standard_normal((16, 41)) * 2
    out["pred_mu"], out["pred_sigma"], out["pred_feats"] = mu, sigma, feats
    out["pred_out"] = np.array([m.predict(f)[0] for f in feats])
    out["pred_z"] = np.array([m.predict(f)[1] for f in feats])
    np.savez_compressed(os.path.join(OUT, "reference_small.npz"), **out)
    print("wrote", os.path.join(OUT, "reference_small.npz"))
    budget_golden(ref, out, l_sink, l_cpu, l_local)


def budget_golden(ref, small, l_sink, l_cpu, l_local):
    """Output-aware budget oracle (budget_oracle.cpp:37-172) on the same
    workload: o_full per head (cache_attention), the step normalizer, the
    streaming label and min_budget at every label granularity for three tau,
    and fit_curve -- all from the compiled reference."""
    seg = (l_sink, l_cpu, l_local, 1)
    q = small["q"]
    H, D = q.shape
    o_full = np.array([ref.cache_attention(small[f"k{h // 4}"], small[f"v{h // 4}"], seg, q[h])
                       for h in range(H)])
    norm = ref.max_output_norm(o_full)
    out = {"o_full": o_full, "normalizer": np.array(norm)}
    taus = (0.05, 0.10, 0.20)
    out["taus"] = np.array(taus)
    stream = np.zeros((len(taus), H), np.int32)
    mb = np.zeros((len(taus), H, 5))
    nb = np.zeros((len(taus), H, 5), np.int64)
    sat = np.zeros((len(taus), H, 5), np.int32)
    for ti, tau in enumerate(taus):
        for h in range(H):
            k, v = small[f"k{h // 4}"], small[f"v{h // 4}"]
            stream[ti, h] = ref.label_streaming(k, v, seg, q[h], o_full[h], norm, tau)
            for i, blk in enumerate((1, 16, 32, 64, 128)):
                mb[ti, h, i], nb[ti, h, i], sat[ti, h, i] = ref.min_budget(k, v, seg, q[h], blk,
                                                                           o_full[h], norm, tau)
    out["streaming"], out["min_budget"], out["min_blocks"], out["saturated"] = stream, mb, nb, sat
    fits = [ref.fit_curve([16, 32, 64, 128], mb[1, h, 1:]) for h in range(H)
            if len(set(mb[1, h, 1:].tolist())) >= 1]
    out["fit"] = np.array(fits)
    np.savez_compressed(os.path.join(OUT, "reference_budget.npz"), **out)
    print("wrote", os.path.join(OUT, "reference_budget.npz"))


if __name__ == "__main__":
    main()
