"""ctypes views of the CPU parity checkers.  TEST INFRASTRUCTURE ONLY.

``COracle``  -- oracle/_build/libfxoracle.so, the C restatement (fx_oracle.c).
``RefOracle`` -- oracle/_ref/libfluxref.so, the unmodified reference compiled
                 from /root/reference/proj/src plus oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libfxoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfluxref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle).  The reference part only when
    /root/reference exists (this container); the GPU box uses prebuilt files."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "dropin"]
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


_MODEL_SHAPES = dict(w1=(256, 41), b1=(256,), w2=(384, 256), b2=(384,), w3=(3, 384), b3=(3,),
                     mu=(41,), sigma=(41,))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class COracle:
    """The C restatement of the hot path (see fx_oracle.c for citations)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.fxo_build_metadata.argtypes = [_f32p, _sz, _sz, C.c_int, _f32p, _f32p]
        L.fxo_build_metadata.restype = C.c_int
        L.fxo_block_scores.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _f64p]
        L.fxo_topk_blocks.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _sz, _u32p, C.c_void_p,
                                      C.POINTER(C.c_int)]
        L.fxo_topk_blocks.restype = _sz
        L.fxo_boundary_gap.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _sz]
        L.fxo_boundary_gap.restype = C.c_double
        L.fxo_selection_tokens.argtypes = [_u32p, _sz, C.c_int, _sz, _u32p]
        L.fxo_selection_tokens.restype = _sz
        L.fxo_blocks_for_budget.argtypes = [C.c_double, _sz, C.c_int]
        L.fxo_blocks_for_budget.restype = _sz
        L.fxo_gathered_attention.argtypes = [_f32p, _f32p, _f32p, _sz, C.c_void_p, _sz, _f64p,
                                             C.POINTER(C.c_double)]
        L.fxo_gathered_attention.restype = _sz
        L.fxo_merge_into.argtypes = [_f64p, C.POINTER(C.c_double), C.POINTER(C.c_size_t), _f64p,
                                     C.c_double, _sz, _sz]
        L.fxo_volume.argtypes = [C.c_int, _sz, _f64p, C.c_int]
        L.fxo_volume.restype = C.c_double
        L.fxo_budget_at.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int]
        L.fxo_budget_at.restype = C.c_double
        L.fxo_plan_group.argtypes = [_f64p, _f64p, _i32p, C.c_int, _sz, C.POINTER(C.c_int), _f64p,
                                     C.POINTER(C.c_double), _f64p]
        L.fxo_plan_group.restype = C.c_int
        L.fxo_execute_group.argtypes = [_f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _f32p, C.c_int,
                                        C.c_int, _f64p, _f32p, _f32p, _f64p, _f64p, _u64p]
        L.fxo_predict.argtypes = [_f64p] * 9 + [_f64p, _f64p]
        L.fxo_rng_normals.argtypes = [C.c_uint64, _f32p, _sz]
        L.fxo_make_model.argtypes = [C.c_uint64] + [_f64p] * 6
        seg = [_f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _f32p]
        L.fxo_max_output_norm.argtypes = [_f64p, _sz, _sz]
        L.fxo_max_output_norm.restype = C.c_double
        L.fxo_cache_attention.argtypes = seg + [_f64p]
        L.fxo_cache_attention.restype = C.c_int
        L.fxo_label_streaming.argtypes = seg + [_f64p, C.c_double, C.c_double]
        L.fxo_label_streaming.restype = C.c_int
        L.fxo_min_budget.argtypes = seg + [C.c_int, _f64p, C.c_double, C.c_double,
                                           C.POINTER(C.c_double), C.POINTER(C.c_size_t),
                                           C.POINTER(C.c_int)]
        L.fxo_min_budget.restype = C.c_int
        L.fxo_fit_curve.argtypes = [_i32p, _f64p, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.fxo_fit_curve.restype = C.c_int
        L.fxo_oracle_props.argtypes = seg + [_f64p, C.c_double, C.c_double,
                                             C.POINTER(C.c_double), C.POINTER(C.c_double),
                                             C.POINTER(C.c_int), _f64p]
        L.fxo_oracle_props.restype = C.c_int
        L.fxo_moments.argtypes = [_f64p, _sz, _f64p]
        L.fxo_gpu_output_norm.argtypes = seg
        L.fxo_gpu_output_norm.restype = C.c_double
        L.fxo_prefill_stats.argtypes = [_f32p, _f32p, _sz, _sz, _sz, _sz, _f32p, _f64p, C.c_double,
                                        C.c_int, C.c_int, _f64p]
        L.fxo_decode_features.argtypes = seg + [_f64p, C.c_double, _f64p]
        self.lib = L

    # -- block index ------------------------------------------------------
    def build_metadata(self, k, blk):
        k = _f32(k)
        rows, dim = k.shape
        nblk = (rows + blk - 1) // blk if blk > 0 else 0
        mins = np.zeros((max(nblk, 1), dim), np.float32)
        maxs = np.zeros((max(nblk, 1), dim), np.float32)
        if self.lib.fxo_build_metadata(k, rows, dim, blk, mins, maxs) != 0:
            raise RuntimeError("invalid-granularity: block size must be >= 1")
        return mins[:nblk], maxs[:nblk]

    def block_scores(self, q, mins, maxs):
        mins, maxs = _f32(mins), _f32(maxs)
        out = np.zeros(mins.shape[0], np.float64)
        self.lib.fxo_block_scores(_f32(q), mins, maxs, mins.shape[0], mins.shape[1], out)
        return out

    def topk_blocks(self, q, mins, maxs, k):
        """-> (blocks in selection order, clamped)"""
        mins, maxs = _f32(mins), _f32(maxs)
        nblk = mins.shape[0]
        out = np.zeros(max(min(k, nblk), 1), np.uint32)
        cl = C.c_int(0)
        n = self.lib.fxo_topk_blocks(_f32(q), mins, maxs, nblk, mins.shape[1], k, out, None,
                                     C.byref(cl))
        return out[:n].copy(), bool(cl.value)

    def boundary_gap(self, q, mins, maxs, k):
        mins, maxs = _f32(mins), _f32(maxs)
        return self.lib.fxo_boundary_gap(_f32(q), mins, maxs, mins.shape[0], mins.shape[1], k)

    def selection_tokens(self, blocks, blk, l_cpu):
        blocks = np.ascontiguousarray(blocks, np.uint32)
        out = np.zeros(max(len(blocks) * blk, 1), np.uint32)
        n = self.lib.fxo_selection_tokens(blocks, len(blocks), blk, l_cpu, out)
        return out[:n].copy()

    def blocks_for_budget(self, bgt, l_cpu, blk):
        return self.lib.fxo_blocks_for_budget(bgt, l_cpu, blk)

    # -- attention --------------------------------------------------------
    def gathered_attention(self, q, k, v, idx=None):
        k, v = _f32(k), _f32(v)
        dim = k.shape[1]
        o = np.zeros(dim, np.float64)
        lse = C.c_double(0)
        if idx is None:
            n = self.lib.fxo_gathered_attention(_f32(q), k, v, dim, None, k.shape[0], o,
                                                C.byref(lse))
        else:
            idx = np.ascontiguousarray(idx, np.uint32)
            n = self.lib.fxo_gathered_attention(_f32(q), k, v, dim, idx.ctypes.data, len(idx), o,
                                                C.byref(lse))
        return o, lse.value, n

    def merge(self, acc, part):
        """acc/part = (o, lse, tokens) -> merged triple (attention.cpp:89-104)."""
        o = _f64(acc[0]).copy()
        lse = C.c_double(acc[1])
        tok = C.c_size_t(acc[2])
        self.lib.fxo_merge_into(o, C.byref(lse), C.byref(tok), _f64(part[0]), part[1], part[2],
                                len(o))
        return o, lse.value, tok.value

    # -- selector ---------------------------------------------------------
    def volume(self, blk, l_cpu, budgets):
        b = _f64(budgets)
        return self.lib.fxo_volume(blk, l_cpu, b, len(b))

    def budget_at(self, bgt0, k, streaming, blk):
        return self.lib.fxo_budget_at(bgt0, k, int(streaming), blk)

    def plan_group(self, bgt0, kslope, streaming, l_cpu):
        G = len(bgt0)
        blk = C.c_int(0)
        vol = C.c_double(0)
        budgets = np.zeros(G, np.float64)
        cand = np.zeros(4, np.float64)
        sg = self.lib.fxo_plan_group(_f64(bgt0), _f64(kslope),
                                     np.ascontiguousarray(streaming, np.int32), G, l_cpu,
                                     C.byref(blk), budgets, C.byref(vol), cand)
        return dict(streaming_group=bool(sg), block_size=blk.value,
                    budgets=budgets if not sg else np.zeros(0), volume=vol.value,
                    candidate_volumes=cand)

    def execute_group(self, k, v, seg, queries, blk, budgets, mins=None, maxs=None):
        """execute_task for one group.  seg = (l_sink, l_cpu, l_local, l_new)."""
        k, v = _f32(k), _f32(v)
        dim = k.shape[1]
        l_sink, l_cpu, l_local, l_new = seg
        if mins is None:
            if blk > 0:
                mins, maxs = self.build_metadata(k[l_sink:l_sink + l_cpu], blk)
            else:
                mins = maxs = np.zeros((1, dim), np.float32)
        mins = mins if len(mins) else np.zeros((1, dim), np.float32)
        maxs = maxs if len(maxs) else np.zeros((1, dim), np.float32)
        queries = _f32(queries)
        G = queries.shape[0]
        o = np.zeros((G, dim), np.float64)
        lse = np.zeros(G, np.float64)
        tok = np.zeros(G, np.uint64)
        self.lib.fxo_execute_group(k, v, dim, l_sink, l_cpu, l_local, l_new, queries, G, blk,
                                   _f64(budgets), _f32(mins), _f32(maxs), o, lse, tok)
        return o, lse, tok

    def predict(self, params, raw):
        """params = dict(w1,b1,w2,b2,w3,b3,mu,sigma) -> (out[3], z[3])"""
        out = np.zeros(3)
        z = np.zeros(3)
        p = [_f64(params[n]) for n in ("w1", "b1", "w2", "b2", "w3", "b3", "mu", "sigma")]
        self.lib.fxo_predict(*p, _f64(raw), out, z)
        return out, z

    def make_model(self, seed):
        """make_model(seed) parameters (predictor.cpp:140-148), mu = 0, sigma = 1."""
        p = {n: np.zeros(int(np.prod(sh))) for n, sh in _MODEL_SHAPES.items()}
        self.lib.fxo_make_model(seed, p["w1"], p["b1"], p["w2"], p["b2"], p["w3"], p["b3"])
        p["sigma"][:] = 1.0
        return p

    def normals(self, seed, n):
        out = np.zeros(n, np.float32)
        self.lib.fxo_rng_normals(seed, out, n)
        return out


    # -- output-aware budget oracle (budget_oracle.cpp) ------------------------
    @staticmethod
    def _seg(k, v, seg, q):
        k, v = _f32(k), _f32(v)
        return [k, v, k.shape[1], *seg, _f32(q)]

    def max_output_norm(self, outs):
        outs = _f64(outs)
        return self.lib.fxo_max_output_norm(outs, outs.shape[0], outs.shape[1])

    def cache_attention(self, k, v, seg, q):
        o = np.zeros(np.shape(k)[1], np.float64)
        if self.lib.fxo_cache_attention(*self._seg(k, v, seg, q), o):
            raise RuntimeError("empty-context: cache has no tokens")
        return o

    def label_streaming(self, k, v, seg, q, o_full, normalizer, tau=0.10):
        r = self.lib.fxo_label_streaming(*self._seg(k, v, seg, q), _f64(o_full), normalizer, tau)
        if r < 0:
            raise RuntimeError("degenerate-normalizer: all head outputs are zero")
        return bool(r)

    def min_budget(self, k, v, seg, q, blk, o_full, normalizer, tau=0.10):
        """-> (budget, blocks, saturated)"""
        bud, nb, sat = C.c_double(0), C.c_size_t(0), C.c_int(0)
        r = self.lib.fxo_min_budget(*self._seg(k, v, seg, q), blk, _f64(o_full), normalizer, tau,
                                    C.byref(bud), C.byref(nb), C.byref(sat))
        if r == -1:
            raise RuntimeError("degenerate-normalizer: all head outputs are zero")
        if r:
            raise RuntimeError("invalid-granularity: blk must be >= 1")
        return bud.value, nb.value, bool(sat.value)

    def fit_curve(self, blks, budgets):
        """-> (k, free_intercept, max_abs_residual)"""
        k, a, r = C.c_double(0), C.c_double(0), C.c_double(0)
        if self.lib.fxo_fit_curve(np.ascontiguousarray(blks, np.int32), _f64(budgets), len(blks),
                                  C.byref(k), C.byref(a), C.byref(r)):
            raise RuntimeError("underdetermined: need at least 2 distinct block sizes")
        return k.value, a.value, r.value

    def oracle_props(self, k, v, seg, q, o_full, normalizer, tau=0.10):
        """pipeline.cpp:256-276 for one head -> (bgt0, k, streaming, budgets[5])"""
        b0, ks, st = C.c_double(0), C.c_double(0), C.c_int(0)
        buds = np.zeros(5, np.float64)
        r = self.lib.fxo_oracle_props(*self._seg(k, v, seg, q), _f64(o_full), normalizer, tau,
                                      C.byref(b0), C.byref(ks), C.byref(st), buds)
        if r:
            raise RuntimeError(f"budget oracle error {r}")
        return b0.value, ks.value, bool(st.value), buds


    # -- features (features.cpp) -----------------------------------------------
    STATS_N = 32

    def moments(self, x):
        out = np.zeros(4)
        x = _f64(x)
        self.lib.fxo_moments(x, len(x), out)
        return out

    def gpu_output_norm(self, k, v, seg, q):
        return self.lib.fxo_gpu_output_norm(*self._seg(k, v, seg, q))

    def prefill_stats(self, k, v, seg3, anchor, budget4, cross_anchor, layer, head):
        """prefill_stats (features.cpp:86-157) -> flat record [32 + 3 D]."""
        k, v = _f32(k), _f32(v)
        D = k.shape[1]
        rec = np.zeros(self.STATS_N + 3 * D)
        self.lib.fxo_prefill_stats(k, v, D, *seg3, _f32(anchor), _f64(budget4), cross_anchor,
                                   layer, head, rec)
        return rec

    def decode_features(self, k, v, seg, q, rec, cross_now):
        out = np.zeros(41)
        self.lib.fxo_decode_features(*self._seg(k, v, seg, q), _f64(rec), cross_now, out)
        return out


class RefOracle:
    """The compiled reference (oracle/_ref/libfluxref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_metadata.argtypes = [_f32p, _sz, _sz, C.c_int, _f32p, _f32p]
        L.ref_block_score.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, C.c_int, _sz, _sz,
                                      C.POINTER(C.c_double)]
        L.ref_topk_blocks.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, C.c_int, _sz, _sz, _u32p,
                                      C.POINTER(C.c_size_t), _u32p, C.POINTER(C.c_size_t),
                                      C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_gathered_attention.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _u32p, _sz, _f64p,
                                             C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.ref_segment_attention.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _f64p,
                                            C.POINTER(C.c_double)]
        L.ref_full_attention.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _f64p]
        L.ref_merge_into.argtypes = [_f64p, C.POINTER(C.c_double), C.POINTER(C.c_uint64), _f64p,
                                     C.c_double, C.c_uint64, _sz]
        L.ref_blocks_for_budget.argtypes = [C.c_double, _sz, C.c_int]
        L.ref_blocks_for_budget.restype = _sz
        L.ref_volume.argtypes = [C.c_int, _sz, _f64p, C.c_int]
        L.ref_volume.restype = C.c_double
        L.ref_budget_at.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int]
        L.ref_budget_at.restype = C.c_double
        L.ref_plan_group.argtypes = [_f64p, _f64p, _i32p, C.c_int, _sz, C.POINTER(C.c_int), _f64p,
                                     C.POINTER(C.c_double), _f64p, C.POINTER(C.c_int)]
        L.ref_execute_group.argtypes = [_f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _f32p, C.c_int,
                                        C.c_int, _f64p, _f64p]
        L.ref_default_kv_attention.argtypes = [_f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _f32p,
                                               _f64p, C.POINTER(C.c_double),
                                               C.POINTER(C.c_uint64)]
        L.ref_batch_create.restype = C.c_void_p
        L.ref_batch_destroy.argtypes = [C.c_void_p]
        L.ref_batch_add.argtypes = [C.c_void_p, _f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _f32p,
                                    C.c_int, C.c_int, _f64p, C.POINTER(C.c_double)]
        L.ref_batch_run.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_void_p]
        L.ref_generate.argtypes = [C.c_char_p]
        L.ref_generate.restype = C.c_void_p
        L.ref_workload_destroy.argtypes = [C.c_void_p]
        L.ref_workload_group_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, _f32p, _f32p]
        L.ref_workload_queries.argtypes = [C.c_void_p, C.c_int, C.c_int, _f32p]
        L.ref_workload_new_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, _f32p, _f32p]
        L.ref_workload_archetype.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_make_model.argtypes = [C.c_uint64]
        L.ref_make_model.restype = C.c_void_p
        L.ref_load_model.argtypes = [C.c_char_p]
        L.ref_load_model.restype = C.c_void_p
        L.ref_model_destroy.argtypes = [C.c_void_p]
        L.ref_model_params.argtypes = [C.c_void_p] + [_f64p] * 8
        L.ref_model_set_norms.argtypes = [C.c_void_p, _f64p, _f64p]
        L.ref_save_model.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_predict.argtypes = [C.c_void_p, _f64p, _f64p, _f64p]
        seg = [_f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _f32p]
        L.ref_cache_attention.argtypes = seg + [_f64p]
        L.ref_min_budget.argtypes = seg + [C.c_int, _f64p, C.c_double, C.c_double,
                                           C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_int)]
        L.ref_label_streaming.argtypes = seg + [_f64p, C.c_double, C.c_double, C.POINTER(C.c_int)]
        L.ref_fit_curve.argtypes = [_i32p, _f64p, C.c_int, C.c_double, C.c_int,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
        L.ref_max_output_norm.argtypes = [_f64p, _sz, _sz, C.POINTER(C.c_double)]
        L.ref_features.argtypes = [_f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _f32p, _f64p, C.c_double,
                                   C.c_int, C.c_int, _f32p, C.c_double, _f64p, _f64p]
        L.ref_gpu_output_norm.argtypes = seg
        L.ref_gpu_output_norm.restype = C.c_double
        L.ref_export_trace.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
        L.ref_import_trace.argtypes = [C.c_char_p]
        L.ref_import_trace.restype = C.c_void_p
        self.lib = L

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def build_metadata(self, k, blk):
        k = _f32(k)
        rows, dim = k.shape
        nblk = (rows + blk - 1) // blk if blk > 0 else 0
        mins = np.zeros((max(nblk, 1), dim), np.float32)
        maxs = np.zeros((max(nblk, 1), dim), np.float32)
        self._check(self.lib.ref_build_metadata(k, rows, dim, blk, mins, maxs))
        return mins[:nblk], maxs[:nblk]

    def block_score(self, q, mins, maxs, blk, source_len, block):
        out = C.c_double(0)
        mins, maxs = _f32(mins), _f32(maxs)
        self._check(self.lib.ref_block_score(_f32(q), mins, maxs, mins.shape[0], mins.shape[1],
                                             blk, source_len, block, C.byref(out)))
        return out.value

    def topk_blocks(self, q, mins, maxs, blk, source_len, k):
        """-> dict(blocks, token_indices, clamped, budget_realized)"""
        mins, maxs = _f32(mins), _f32(maxs)
        nblk, dim = mins.shape
        kk = min(k, nblk)
        blocks = np.zeros(max(kk, 1), np.uint32)
        tokens = np.zeros(max(kk * blk, 1), np.uint32)
        nb, nt = C.c_size_t(0), C.c_size_t(0)
        cl, br = C.c_int(0), C.c_double(0)
        self._check(self.lib.ref_topk_blocks(_f32(q), mins, maxs, nblk, dim, blk, source_len, k,
                                             blocks, C.byref(nb), tokens, C.byref(nt),
                                             C.byref(cl), C.byref(br)))
        return dict(blocks=blocks[:nb.value].copy(), token_indices=tokens[:nt.value].copy(),
                    clamped=bool(cl.value), budget_realized=br.value)

    def gathered_attention(self, q, k, v, idx):
        k, v = _f32(k), _f32(v)
        idx = np.ascontiguousarray(idx, np.uint32)
        o = np.zeros(k.shape[1])
        lse = C.c_double(0)
        tok = C.c_uint64(0)
        self._check(self.lib.ref_gathered_attention(_f32(q), k, v, k.shape[0], k.shape[1], idx,
                                                    len(idx), o, C.byref(lse), C.byref(tok)))
        return o, lse.value, tok.value

    def segment_attention(self, q, k, v):
        k, v = _f32(k), _f32(v)
        o = np.zeros(k.shape[1])
        lse = C.c_double(0)
        self._check(self.lib.ref_segment_attention(_f32(q), k, v, k.shape[0], k.shape[1], o,
                                                   C.byref(lse)))
        return o, lse.value

    def full_attention(self, q, k, v):
        k, v = _f32(k), _f32(v)
        o = np.zeros(k.shape[1])
        self._check(self.lib.ref_full_attention(_f32(q), k, v, k.shape[0], k.shape[1], o))
        return o

    def merge(self, acc, part):
        o = _f64(acc[0]).copy()
        lse = C.c_double(acc[1])
        tok = C.c_uint64(acc[2])
        self._check(self.lib.ref_merge_into(o, C.byref(lse), C.byref(tok), _f64(part[0]), part[1],
                                            part[2], len(o)))
        return o, lse.value, tok.value

    def blocks_for_budget(self, bgt, l_cpu, blk):
        return self.lib.ref_blocks_for_budget(bgt, l_cpu, blk)

    def volume(self, blk, l_cpu, budgets):
        b = _f64(budgets)
        return self.lib.ref_volume(blk, l_cpu, b, len(b))

    def budget_at(self, bgt0, k, streaming, blk):
        return self.lib.ref_budget_at(bgt0, k, int(streaming), blk)

    def plan_group(self, bgt0, kslope, streaming, l_cpu):
        G = len(bgt0)
        blk, sg = C.c_int(0), C.c_int(0)
        vol = C.c_double(0)
        budgets = np.zeros(max(G, 1))
        cand = np.zeros(4)
        self._check(self.lib.ref_plan_group(_f64(bgt0), _f64(kslope),
                                            np.ascontiguousarray(streaming, np.int32), G, l_cpu,
                                            C.byref(blk), budgets, C.byref(vol), cand,
                                            C.byref(sg)))
        return dict(streaming_group=bool(sg.value), block_size=blk.value,
                    budgets=budgets[:G] if not sg.value else np.zeros(0), volume=vol.value,
                    candidate_volumes=cand)

    def execute_group(self, k, v, seg, queries, blk, budgets):
        k, v = _f32(k), _f32(v)
        queries = _f32(queries)
        G, dim = queries.shape
        o = np.zeros((G, dim))
        self._check(self.lib.ref_execute_group(k, v, dim, *seg, queries, G, blk, _f64(budgets),
                                               o))
        return o

    def default_kv_attention(self, k, v, seg, q):
        k, v = _f32(k), _f32(v)
        o = np.zeros(k.shape[1])
        lse = C.c_double(0)
        tok = C.c_uint64(0)
        self._check(self.lib.ref_default_kv_attention(k, v, k.shape[1], *seg, _f32(q), o,
                                                      C.byref(lse), C.byref(tok)))
        return o, lse.value, tok.value

    # -- output-aware budget oracle (budget_oracle.cpp) -------------------
    def cache_attention(self, k, v, seg, q):
        k, v = _f32(k), _f32(v)
        o = np.zeros(k.shape[1])
        self._check(self.lib.ref_cache_attention(k, v, k.shape[1], *seg, _f32(q), o))
        return o

    def min_budget(self, k, v, seg, q, blk, o_full, normalizer, tau=0.10):
        k, v = _f32(k), _f32(v)
        bud, nb, sat = C.c_double(0), C.c_uint64(0), C.c_int(0)
        self._check(self.lib.ref_min_budget(k, v, k.shape[1], *seg, _f32(q), blk, _f64(o_full),
                                            normalizer, tau, C.byref(bud), C.byref(nb),
                                            C.byref(sat)))
        return bud.value, nb.value, bool(sat.value)

    def label_streaming(self, k, v, seg, q, o_full, normalizer, tau=0.10):
        k, v = _f32(k), _f32(v)
        st = C.c_int(0)
        self._check(self.lib.ref_label_streaming(k, v, k.shape[1], *seg, _f32(q), _f64(o_full),
                                                 normalizer, tau, C.byref(st)))
        return bool(st.value)

    def fit_curve(self, blks, budgets, bgt0=0.0, streaming=False):
        k, a, r = C.c_double(0), C.c_double(0), C.c_double(0)
        self._check(self.lib.ref_fit_curve(np.ascontiguousarray(blks, np.int32), _f64(budgets),
                                           len(blks), bgt0, int(streaming), C.byref(k),
                                           C.byref(a), C.byref(r)))
        return k.value, a.value, r.value

    def max_output_norm(self, outs):
        outs = _f64(outs)
        out = C.c_double(0)
        self._check(self.lib.ref_max_output_norm(outs, outs.shape[0], outs.shape[1], C.byref(out)))
        return out.value

    def features(self, k, v, seg, anchor, budget4, cross_anchor, layer, head, q, cross_now):
        """prefill_stats (no decoded rows) + decode_features -> (record, features[41])."""
        k, v = _f32(k), _f32(v)
        D = k.shape[1]
        rec = np.zeros(32 + 3 * D)
        f = np.zeros(41)
        self._check(self.lib.ref_features(k, v, D, *seg, _f32(anchor), _f64(budget4), cross_anchor,
                                          layer, head, _f32(q), cross_now, rec, f))
        return rec, f

    def gpu_output_norm(self, k, v, seg, q):
        k, v = _f32(k), _f32(v)
        return self.lib.ref_gpu_output_norm(k, v, k.shape[1], *seg, _f32(q))

    def export_trace(self, workload, path, input_hash=0):
        self._check(self.lib.ref_export_trace(workload.h, path.encode(), input_hash))

    def import_trace(self, path, **spec):
        """import_trace -> a workload handle (spec gives the accessor shapes)."""
        h = self.lib.ref_import_trace(path.encode())
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return _RefWorkload(self, h, spec)

    # -- executed scheduler (CPU baseline) -------------------------------
    def batch(self):
        return _RefBatch(self)

    # -- workload generator ------------------------------------------------
    def generate(self, **spec):
        h = self.lib.ref_generate(json.dumps(spec).encode())
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return _RefWorkload(self, h, spec)

    # -- predictor ----------------------------------------------------------
    def make_model(self, seed):
        return _RefModel(self, self.lib.ref_make_model(seed))

    def load_model(self, path):
        h = self.lib.ref_load_model(path.encode())
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return _RefModel(self, h)


class _RefBatch:
    def __init__(self, ref):
        self.ref = ref
        self.h = ref.lib.ref_batch_create()
        self.groups = []

    def add(self, k, v, seg, queries, blk, budgets):
        k, v, queries = _f32(k), _f32(v), _f32(queries)
        ms = C.c_double(0)
        self.ref._check(self.ref.lib.ref_batch_add(self.h, k, v, k.shape[1], *seg, queries,
                                                   queries.shape[0], blk, _f64(budgets),
                                                   C.byref(ms)))
        self.groups.append(queries.shape)
        return ms.value

    def run(self, host_workers, want_outputs=False):
        sec = C.c_double(0)
        out = None
        if want_outputs:
            G, dim = self.groups[0]
            out = np.zeros((len(self.groups), G, dim))
        self.ref._check(self.ref.lib.ref_batch_run(self.h, host_workers, C.byref(sec),
                                                   out.ctypes.data if out is not None else None))
        return sec.value, out

    def __del__(self):
        try:
            self.ref.lib.ref_batch_destroy(self.h)
        except Exception:
            pass


class _RefWorkload:
    def __init__(self, ref, h, spec):
        self.ref, self.h, self.spec = ref, h, spec
        self.heads = spec.get("heads", 8)
        self.group_size = spec.get("group_size", 4)
        self.head_dim = spec.get("head_dim", 64)
        self.context_len = spec.get("context_len", 4096)
        self.sink = spec.get("sink_tokens", 64)
        self.local = spec.get("local_tokens", 256)

    def group_kv(self, layer, g):
        n = self.context_len * self.head_dim
        k = np.zeros(n, np.float32)
        v = np.zeros(n, np.float32)
        self.ref._check(self.ref.lib.ref_workload_group_kv(self.h, layer, g, k, v))
        return k.reshape(self.context_len, self.head_dim), v.reshape(self.context_len,
                                                                     self.head_dim)

    def queries(self, layer, step):
        out = np.zeros(self.heads * self.head_dim, np.float32)
        self.ref._check(self.ref.lib.ref_workload_queries(self.h, layer, step, out))
        return out.reshape(self.heads, self.head_dim)

    def new_kv(self, layer, step):
        groups = self.heads // self.group_size
        k = np.zeros(groups * self.head_dim, np.float32)
        v = np.zeros(groups * self.head_dim, np.float32)
        self.ref._check(self.ref.lib.ref_workload_new_kv(self.h, layer, step, k, v))
        return k.reshape(groups, self.head_dim), v.reshape(groups, self.head_dim)

    def archetype(self, layer, head):
        return self.ref.lib.ref_workload_archetype(self.h, layer, head)

    def __del__(self):
        try:
            self.ref.lib.ref_workload_destroy(self.h)
        except Exception:
            pass


class _RefModel:
    SHAPES = dict(w1=(256, 41), b1=(256,), w2=(384, 256), b2=(384,), w3=(3, 384), b3=(3,),
                  mu=(41,), sigma=(41,))

    def __init__(self, ref, h):
        self.ref, self.h = ref, h

    def params(self):
        p = {n: np.zeros(int(np.prod(s))) for n, s in self.SHAPES.items()}
        self.ref._check(self.ref.lib.ref_model_params(self.h, *[p[n] for n in self.SHAPES]))
        return p

    def set_norms(self, mu, sigma):
        self.ref._check(self.ref.lib.ref_model_set_norms(self.h, _f64(mu), _f64(sigma)))

    def save(self, path):
        self.ref._check(self.ref.lib.ref_save_model(self.h, path.encode()))

    def predict(self, raw):
        out = np.zeros(3)
        z = np.zeros(3)
        self.ref._check(self.ref.lib.ref_predict(self.h, _f64(raw), out, z))
        return out, z

    def __del__(self):
        try:
            self.ref.lib.ref_model_destroy(self.h)
        except Exception:
            pass
