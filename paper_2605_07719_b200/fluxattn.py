"""Python view of the B200 hot path, mirroring the reference operator API.

Reference interface (``/root/reference/proj/include/fluxattn``):
``build_metadata`` / ``block_score`` / ``topk_blocks`` / ``sparse_attention`` /
``blocks_for_budget`` (block_index.hpp:41-56), ``segment_attention`` /
``full_attention`` / ``merge_partials`` / ``combine_partials`` /
``default_kv_attention`` (attention.hpp:26-70), ``volume`` / ``budget_at`` /
``plan_group`` / ``priority`` (selector.hpp:28-39), ``execute_task``
(scheduler.hpp:128).  Names, argument meaning and error codes follow the
reference; every computation runs in the CUDA library through the C-ABI
(``_native``).  torch is used only to own device memory and streams.

``SparseDecoder`` is the batched, device-resident production path (one call
per decode step for a whole batch), the analog of the reference's
``run(queue, profile, RunMode::Executed)`` over ``execute_task``.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from ._native import LIB, check

CANDIDATE_BLOCKS = (16, 32, 64, 128)  # selector.hpp:12


# ---------------------------------------------------------------------------
# reference data types (block_index.hpp:16-39, attention.hpp:17-23,
# selector.hpp:16-23, budget_oracle.hpp:17-21, scheduler.hpp:31-43, 123-126)
# ---------------------------------------------------------------------------
@dataclass
class BlockMetadata:
    block_size: int
    source_len: int
    dim: int
    block_count: int
    mins: np.ndarray  # [block_count x dim] f32
    maxs: np.ndarray
    _dev: Optional[torch.Tensor] = None  # [nblk][2][dim] device copy

    def block_begin(self, b: int) -> int:
        return b * self.block_size

    def block_end(self, b: int) -> int:
        return min(self.source_len, (b + 1) * self.block_size)


@dataclass
class SelectionResult:
    block_size: int = 0
    source_len: int = 0
    blocks: List[int] = field(default_factory=list)
    token_indices: List[int] = field(default_factory=list)
    budget_realized: float = 0.0
    clamped: bool = False


@dataclass
class PartialOutput:
    o: np.ndarray = field(default_factory=lambda: np.zeros(0))
    lse: float = -math.inf
    tokens: int = 0

    def empty(self) -> bool:
        return self.tokens == 0


@dataclass
class HeadProperties:
    bgt0: float = 0.0
    k: float = 0.0
    streaming: bool = False


@dataclass
class GroupPlan:
    group_id: int = 0
    block_size: int = 0
    budgets: List[float] = field(default_factory=list)
    volume: float = 0.0
    streaming_group: bool = False
    candidate_volumes: List[float] = field(default_factory=lambda: [0.0] * 4)


@dataclass
class SegmentedKvCache:
    """Position-ordered segments sink | cpu | local | new (kv_cache.hpp:13-18)."""

    k_sink: np.ndarray
    v_sink: np.ndarray
    k_cpu: np.ndarray
    v_cpu: np.ndarray
    k_local: np.ndarray
    v_local: np.ndarray
    k_new: np.ndarray = None
    v_new: np.ndarray = None

    def __post_init__(self):
        d = self.dim()
        if self.k_new is None:
            self.k_new = np.zeros((0, d), np.float32)
            self.v_new = np.zeros((0, d), np.float32)
        for kk, vv in self._pairs():
            if kk.shape[0] != vv.shape[0]:
                raise RuntimeError("bad-shape: K/V row count differs in a segment")
            if kk.shape[0] and (kk.shape[1] != d or vv.shape[1] != d):
                raise RuntimeError("bad-shape: segment dim mismatch")
            if kk.size and (not np.isfinite(kk).all() or not np.isfinite(vv).all()):
                raise RuntimeError("non-finite: cache tensor")

    def _pairs(self):
        return [(self.k_sink, self.v_sink), (self.k_cpu, self.v_cpu),
                (self.k_local, self.v_local), (self.k_new, self.v_new)]

    def dim(self) -> int:
        for kk in (self.k_sink, self.k_cpu, self.k_local, self.k_new):
            if kk is not None and kk.ndim == 2 and kk.shape[0] > 0:
                return kk.shape[1]
        return 0

    def lens(self):
        return (len(self.k_sink), len(self.k_cpu), len(self.k_local), len(self.k_new))

    def append_new(self, k: np.ndarray, v: np.ndarray) -> None:
        if not (np.isfinite(k).all() and np.isfinite(v).all()):
            raise RuntimeError("non-finite: appended kv row")
        self.k_new = np.vstack([self.k_new, np.asarray(k, np.float32)[None]])
        self.v_new = np.vstack([self.v_new, np.asarray(v, np.float32)[None]])

    def stacked(self):
        """K, V in position order, [total x dim] f32."""
        k = np.vstack([a for a, _ in self._pairs() if len(a)]).astype(np.float32)
        v = np.vstack([b for _, b in self._pairs() if len(b)]).astype(np.float32)
        return k, v


@dataclass
class SparseTask:
    group_id: int
    plan: GroupPlan
    cache: SegmentedKvCache
    metadata: BlockMetadata
    queries: List[np.ndarray]


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _finite(x) -> bool:
    return bool(np.isfinite(np.asarray(x)).all())


# ---------------------------------------------------------------------------
# engine: one CUDA context (device + stream) behind the C-ABI
# ---------------------------------------------------------------------------
class Engine:
    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("no-device: the fluxattn B200 path needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        h = C.c_void_p()
        check(LIB.fx_ctx_create(device, C.byref(h)))
        self.ctx = h
        self.sync_stream()

    def sync_stream(self):
        """Run our kernels on torch's current stream of this device."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        check(LIB.fx_ctx_set_stream(self.ctx, C.c_void_p(s)))

    def launches(self) -> int:
        return int(LIB.fx_ctx_launches(self.ctx))

    def synchronize(self) -> None:
        """Wait for the ctx stream; raises device-detected argument errors
        (e.g. invalid-granularity from a device-resident given plan)."""
        check(LIB.fx_ctx_synchronize(self.ctx))

    def close(self):
        if getattr(self, "ctx", None):
            LIB.fx_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers ------------------------------------------------------------
    def _dev(self, a, dtype=torch.float32) -> torch.Tensor:
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(self.device)

    # -- block index (block_index.hpp:41-56) ---------------------------------
    def build_metadata(self, k_cpu: np.ndarray, block_size: int) -> BlockMetadata:
        """build_metadata (block_index.cpp:10-39)."""
        if block_size <= 0:
            raise RuntimeError("invalid-granularity: block size must be >= 1")
        k_cpu = np.ascontiguousarray(k_cpu, np.float32)
        rows, dim = k_cpu.shape if k_cpu.ndim == 2 else (0, 0)
        nblk = (rows + block_size - 1) // block_size
        dev = torch.empty((max(nblk, 1), 2, max(dim, 1)), dtype=torch.float32, device=self.device)
        if nblk:
            kd = self._dev(k_cpu)
            check(LIB.fx_build_metadata(self.ctx, _ptr(kd), N.FX_F32, rows, dim, block_size,
                                        _ptr(dev)))
        h = dev[:nblk].cpu().numpy()
        return BlockMetadata(block_size, rows, dim, nblk, h[:, 0, :dim].copy(),
                             h[:, 1, :dim].copy(), dev[:nblk])

    def _meta_dev(self, meta: BlockMetadata) -> torch.Tensor:
        if meta._dev is None:
            m = np.stack([meta.mins, meta.maxs], axis=1)
            meta._dev = self._dev(m)
        return meta._dev

    def block_scores(self, q: np.ndarray, meta: BlockMetadata) -> np.ndarray:
        out = torch.empty(max(meta.block_count, 1), dtype=torch.float64, device=self.device)
        qd = self._dev(q)
        check(LIB.fx_block_scores(self.ctx, _ptr(qd), _ptr(self._meta_dev(meta)), N.FX_F32,
                                  meta.block_count, meta.dim, _ptr(out)))
        return out[:meta.block_count].cpu().numpy()

    def block_score(self, q: np.ndarray, meta: BlockMetadata, block: int) -> float:
        """block_score (block_index.cpp:41-53)."""
        if block >= meta.block_count or block < 0:
            raise RuntimeError("bad-block: block id out of range")
        return float(self.block_scores(q, meta)[block])

    def topk_blocks(self, q: np.ndarray, meta: BlockMetadata, k: int) -> SelectionResult:
        """topk_blocks (block_index.cpp:55-83)."""
        sel = SelectionResult(block_size=meta.block_size, source_len=meta.source_len)
        out = torch.empty(max(min(k, meta.block_count), 1), dtype=torch.int32, device=self.device)
        ke, cl = C.c_int64(0), C.c_int32(0)
        qd = self._dev(q)
        check(LIB.fx_topk_blocks(self.ctx, _ptr(qd), _ptr(self._meta_dev(meta)), N.FX_F32,
                                 meta.block_count, meta.dim, k, _ptr(out), C.byref(ke),
                                 C.byref(cl)))
        sel.clamped = bool(cl.value)
        if ke.value == 0:
            return sel
        sel.blocks = [int(x) for x in out[:ke.value].cpu().numpy().view(np.uint32)]
        toks = []
        for b in sel.blocks:
            toks.extend(range(meta.block_begin(b), meta.block_end(b)))
        sel.token_indices = sorted(toks)
        sel.budget_realized = (len(sel.token_indices) / meta.source_len) if meta.source_len else 0.0
        return sel

    def blocks_for_budget(self, budget: float, l_cpu: int, block_size: int) -> int:
        """blocks_for_budget (block_index.cpp:96-103), evaluated on device."""
        b = self._dev(np.array([budget]), torch.float64)
        blk = self._dev(np.array([block_size]), torch.int32)
        out = torch.zeros(1, dtype=torch.int32, device=self.device)
        check(LIB.fx_blocks_for_budget(self.ctx, 1, _ptr(b), _ptr(blk), l_cpu, _ptr(out)))
        return int(out.item())

    # -- attention (attention.hpp:26-70) --------------------------------------
    def gathered_attention(self, q, k, v, idx) -> PartialOutput:
        """detail::gathered_attention_unchecked (attention.cpp:57-87)."""
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        idx = np.ascontiguousarray(idx, np.uint32)
        dim = k.shape[1]
        o = torch.empty(dim, dtype=torch.float32, device=self.device)
        lse = torch.empty(1, dtype=torch.float32, device=self.device)
        if len(idx) == 0:
            return PartialOutput()
        kd, vd, qd = self._dev(k), self._dev(v), self._dev(q)
        idd = torch.as_tensor(idx.view(np.int32)).to(self.device)
        check(LIB.fx_gathered_attention(self.ctx, _ptr(qd), _ptr(kd), _ptr(vd), N.FX_F32,
                                        k.shape[0], dim, _ptr(idd), len(idx), _ptr(o), _ptr(lse)))
        return PartialOutput(o.double().cpu().numpy(), float(lse.item()), len(idx))

    def segment_attention(self, q, k, v) -> PartialOutput:
        """segment_attention (attention.cpp:111-116)."""
        k = np.asarray(k, np.float32)
        v = np.asarray(v, np.float32)
        if len(k) == 0 or len(v) == 0:
            raise RuntimeError("empty-context: attention over zero keys")
        if len(k) != len(v):
            raise RuntimeError("bad-shape: K/V row count mismatch")
        if len(q) != k.shape[1]:
            raise RuntimeError("bad-shape: query width != key width")
        if not (_finite(q) and _finite(k) and _finite(v)):
            raise RuntimeError("non-finite: attention input")
        return self.gathered_attention(q, k, v, np.arange(len(k)))

    def full_attention(self, q, k, v) -> np.ndarray:
        return self.segment_attention(q, k, v).o

    def combine_partials(self, parts: Sequence[PartialOutput]) -> PartialOutput:
        """combine_partials (attention.cpp:118-122): LSE merge on device."""
        live = [p for p in parts if not p.empty()]
        if not live:
            return PartialOutput()
        dim = len(live[0].o)
        op = self._dev(np.stack([p.o for p in live]))
        lp = self._dev(np.array([p.lse for p in live]))
        o = torch.empty(dim, dtype=torch.float32, device=self.device)
        lse = torch.empty(1, dtype=torch.float32, device=self.device)
        check(LIB.fx_merge_partials(self.ctx, len(live), dim, _ptr(op), _ptr(lp), _ptr(o),
                                    _ptr(lse)))
        return PartialOutput(o.double().cpu().numpy(), float(lse.item()),
                             sum(p.tokens for p in live))

    def merge_partials(self, parts: Sequence[PartialOutput]) -> np.ndarray:
        acc = self.combine_partials(parts)
        if acc.empty():
            raise RuntimeError("empty-context: all partials empty")
        return acc.o

    def default_kv_attention(self, q, cache: SegmentedKvCache) -> PartialOutput:
        """default_kv_attention (attention.cpp:143-151): sink + local + new."""
        k, v = cache.stacked()
        ls, lc, ll, ln = cache.lens()
        idx = np.concatenate([np.arange(ls), np.arange(ls + lc, ls + lc + ll + ln)])
        return self.gathered_attention(q, k, v, idx)

    def sparse_attention(self, q, cache: SegmentedKvCache, sel: SelectionResult) -> PartialOutput:
        """sparse_attention (block_index.cpp:85-94)."""
        if sel.source_len != len(cache.k_cpu):
            raise RuntimeError("stale-selection: cpu segment length changed")
        if not sel.token_indices:
            return PartialOutput()
        if not _finite(q):
            raise RuntimeError("non-finite: query")
        return self.gathered_attention(q, cache.k_cpu, cache.v_cpu, np.asarray(sel.token_indices))

    # -- selector (selector.hpp:28-39) ----------------------------------------
    def plan_groups(self, props: Sequence[Sequence[HeadProperties]], l_cpu: int) -> List[GroupPlan]:
        """plan_group for many groups in one device launch (selector.cpp:21-46)."""
        n = len(props)
        G = len(props[0]) if n else 0
        if n == 0:
            return []
        if G == 0:
            raise RuntimeError("empty-group: plan_group needs at least one head")
        b0 = self._dev(np.array([[p.bgt0 for p in g] for g in props]), torch.float64)
        ks = self._dev(np.array([[p.k for p in g] for g in props]), torch.float64)
        st = self._dev(np.array([[int(p.streaming) for p in g] for g in props]), torch.int32)
        blk = torch.zeros(n, dtype=torch.int32, device=self.device)
        bud = torch.zeros((n, G), dtype=torch.float64, device=self.device)
        vol = torch.zeros(n, dtype=torch.float64, device=self.device)
        cand = torch.zeros((n, 4), dtype=torch.float64, device=self.device)
        check(LIB.fx_plan_groups(self.ctx, n, G, l_cpu, _ptr(b0), _ptr(ks), _ptr(st), _ptr(blk),
                                 _ptr(bud), _ptr(vol), _ptr(cand), None))
        blk, bud, vol, cand = (t.cpu().numpy() for t in (blk, bud, vol, cand))
        out = []
        for i in range(n):
            sg = int(blk[i]) == 0
            out.append(GroupPlan(group_id=i, block_size=int(blk[i]),
                                 budgets=[] if sg else [float(x) for x in bud[i]],
                                 volume=float(vol[i]), streaming_group=sg,
                                 candidate_volumes=[float(x) for x in cand[i]]))
        return out

    def plan_group(self, group_id: int, props: Sequence[HeadProperties], l_cpu: int) -> GroupPlan:
        if len(props) == 0:
            raise RuntimeError("empty-group: plan_group needs at least one head")
        p = self.plan_groups([props], l_cpu)[0]
        p.group_id = group_id
        return p

    @staticmethod
    def priority(plan: GroupPlan) -> float:
        if plan.streaming_group:
            raise RuntimeError("not-schedulable: streaming group has no priority")
        return plan.volume

    # -- execute_task (scheduler.cpp:78-96) -------------------------------------
    def execute_task(self, task: SparseTask) -> List[np.ndarray]:
        """One group through the batched device path (B = 1, Hkv = 1)."""
        if task.cache is None or task.metadata is None:
            raise RuntimeError("no-context: task has no executable payload")
        cache = task.cache
        ls, lc, ll, ln = cache.lens()
        G = len(task.queries)
        D = cache.dim()
        dec = SparseDecoder(self, batch=1, kv_heads=1, group_size=G, head_dim=D,
                            l_sink=ls, l_cpu=lc, l_local=ll, max_new=max(ln, 1),
                            dtype="f32")
        k, v = cache.stacked()
        dec.load_group(0, 0, k, v)
        dec.l_new = ln
        dec.build_metadata()
        q = np.stack(task.queries).astype(np.float32)[None]
        o, _ = dec.step(q, blk=[[task.plan.block_size]], budgets=[[list(task.plan.budgets)]])
        return [o[0, h].astype(np.float64) for h in range(G)]


# ---------------------------------------------------------------------------
# batched production path
# ---------------------------------------------------------------------------
class SparseDecoder:
    """Device-resident KV for a batch and the one-call-per-step decode.

    K and V: [batch][kv_heads][l_cap][head_dim] (bf16 or f32) with rows
    sink | cpu | local | decoded; metadata at all four candidate granularities
    is built once (K1) and kept resident, like the reference's memo
    (pipeline.cpp:208-218).
    """

    def __init__(self, engine: Engine, batch: int, kv_heads: int, group_size: int,
                 head_dim: int, l_sink: int, l_cpu: int, l_local: int, max_new: int = 64,
                 dtype: str = "bf16", k: torch.Tensor = None, v: torch.Tensor = None):
        self.eng = engine
        self.dtype = dtype
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.tdtype = tdt
        self.lay = N.Layout(batch, kv_heads, group_size, head_dim,
                            N.FX_BF16 if dtype == "bf16" else N.FX_F32, 0, l_sink, l_cpu,
                            l_local, SparseDecoder.cap_rows(l_sink + l_cpu + l_local, max_new))
        shape = (batch, kv_heads, self.lay.l_cap, head_dim)
        dev = engine.device
        self.k = k if k is not None else torch.zeros(shape, dtype=tdt, device=dev)
        self.v = v if v is not None else torch.zeros(shape, dtype=tdt, device=dev)
        assert tuple(self.k.shape) == shape and self.k.dtype == tdt
        self.meta = []
        for blk in CANDIDATE_BLOCKS:
            nb = max(1, (l_cpu + blk - 1) // blk)
            self.meta.append(torch.empty((batch, kv_heads, nb, 2, head_dim), dtype=tdt, device=dev))
        self.absmax = torch.zeros((batch, kv_heads, head_dim), dtype=torch.float32, device=dev)
        self.l_new = 0
        H = kv_heads * group_size
        self.heads = H
        self.nblk16 = max(1, (l_cpu + 15) // 16)
        self.sel_words = (self.nblk16 + 31) // 32
        self.plan_blk = torch.zeros((batch, kv_heads), dtype=torch.int32, device=dev)
        self.plan_budgets = torch.zeros((batch, H), dtype=torch.float64, device=dev)
        self.plan_volume = torch.zeros((batch, kv_heads), dtype=torch.float64, device=dev)
        self.plan_cand = torch.zeros((batch, kv_heads, 4), dtype=torch.float64, device=dev)
        self.plan_kblocks = torch.zeros((batch, H), dtype=torch.int32, device=dev)
        self.sel_bits = torch.zeros((batch, H, self.sel_words), dtype=torch.int32, device=dev)
        self.o = torch.empty((batch, H, head_dim), dtype=torch.float32, device=dev)
        self.lse = torch.empty((batch, H), dtype=torch.float32, device=dev)
        self.args = N.StepArgs()
        # context-parallel shard (context_parallel.py): whole-sequence cpu
        # length for the plan and this shard's first global cpu row
        self.l_cpu_total = 0
        self.cpu_offset = 0

    @staticmethod
    def cap_rows(context: int, max_new: int) -> int:
        """Rows per (b, g): context + decode room, rounded up to a multiple of 16
        so every (b, g) starts on a 16-row TMA unit."""
        return (context + max_new + 15) // 16 * 16

    # -- data --------------------------------------------------------------
    def load_group(self, b: int, g: int, k: np.ndarray, v: np.ndarray) -> None:
        """Copy one group's position-ordered K/V ([rows x D] f32) into the cache."""
        n = k.shape[0]
        self.k[b, g, :n] = torch.as_tensor(np.ascontiguousarray(k)).to(self.k.device, self.tdtype)
        self.v[b, g, :n] = torch.as_tensor(np.ascontiguousarray(v)).to(self.v.device, self.tdtype)

    def build_metadata(self, means: bool = False) -> None:
        """K1 over every (b, g): levels 16/32/64/128 + absmax (one launch);
        means=True also writes the per-block mean keys self.means[i]
        [B][Hkv][nblk][D] f32 (north-star item 1)."""
        if self.lay.l_cpu == 0:
            return
        if not means:
            check(LIB.fx_build_metadata_levels(self.eng.ctx, C.byref(self.lay), _ptr(self.k),
                                               *[_ptr(m) for m in self.meta], _ptr(self.absmax)))
            return
        lay = self.lay
        self.means = [torch.empty((lay.batch, lay.kv_heads, m.shape[2], lay.head_dim), dtype=torch.float32,
                                  device=self.eng.device) for m in self.meta]
        lv = (C.c_void_p * 4)(*[m.data_ptr() for m in self.meta])
        mv = (C.c_void_p * 4)(*[m.data_ptr() for m in self.means])
        check(LIB.fx_build_metadata_means(self.eng.ctx, C.byref(lay), _ptr(self.k), lv, _ptr(self.absmax), mv))

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor) -> None:
        """append_new (kv_cache.hpp:68-73) for every group: [B][Hkv][D] f32 device."""
        row = self.lay.l_sink + self.lay.l_cpu + self.lay.l_local + self.l_new
        check(LIB.fx_append_kv(self.eng.ctx, C.byref(self.lay), _ptr(self.k), _ptr(self.v), row,
                               _ptr(k_new.float().contiguous()), _ptr(v_new.float().contiguous())))
        self.l_new += 1

    # -- one decode step ------------------------------------------------------
    def step(self, q, props=None, fixed=None, full=False, blk=None, budgets=None,
             out: torch.Tensor = None, lse: torch.Tensor = None, sel_in: torch.Tensor = None,
             append=None):
        """Plan -> select -> attend+merge for every head of the batch.

        q: [B][H][D] f32 (device tensor or host array).  Budget source, one of:
          props = (bgt0, kslope, streaming) device tensors [B][H]  (selector)
          fixed = (blk, bgt)                                      (pipeline.cpp:304-311)
          full  = True                                            (pipeline.cpp:298-303)
          blk = [B][Hkv], budgets = [B][H]                        (given plan)
          blk = "keep"                        (given plan = the last step's plan)
        sel_in: a given selection [B][H][sel_words] (skips score/select;
        needs a given plan) -- the context-parallel attend phase.
        append: (k_new, v_new) [B][Hkv][D] f32 device rows appended as decoded row
        l_new inside the step's first kernel (the previous step's token; saves the
        separate append launch); the step then attends them.
        Returns (o [B][H][D] f32, lse [B][H]) as device tensors when q is a
        device tensor, else numpy arrays.
        """
        host = not isinstance(q, torch.Tensor)
        qd = torch.as_tensor(np.ascontiguousarray(q, np.float32)).to(self.eng.device) if host else q
        a = self._args(qd, props, fixed, full, blk, budgets)
        a.sel_in = None if sel_in is None else sel_in.data_ptr()
        if append is not None:
            self._append = [t.float().contiguous() for t in append]
            a.append_k, a.append_v = (t.data_ptr() for t in self._append)
        res = self._finish(a, host, out, lse)
        if append is not None:
            self.l_new += 1
        return res

    def _args(self, qd, props, fixed, full, blk, budgets) -> N.StepArgs:
        a = self.args
        a.k, a.v = self.k.data_ptr(), self.v.data_ptr()
        for i, m in enumerate(self.meta):
            a.meta[i] = m.data_ptr()
        a.absmax = self.absmax.data_ptr()
        a.l_new = self.l_new
        a.q = qd.data_ptr()
        a.l_cpu_total = self.l_cpu_total
        a.cpu_offset = self.cpu_offset
        a.sel_in = None
        a.append_k = a.append_v = None
        a.bgt0 = a.kslope = a.streaming = None
        if props is not None:
            a.plan_mode = N.FX_PLAN_PROPS
            self._props = [t.contiguous() for t in props]
            a.bgt0, a.kslope, a.streaming = (t.data_ptr() for t in self._props)
        elif fixed is not None:
            a.plan_mode = N.FX_PLAN_FIXED
            a.fixed_block_size, a.fixed_budget = int(fixed[0]), float(fixed[1])
        elif full:
            a.plan_mode = N.FX_PLAN_FULL
        elif isinstance(blk, str) and blk == "keep":
            a.plan_mode = N.FX_PLAN_GIVEN
        else:
            a.plan_mode = N.FX_PLAN_GIVEN
            bk = np.asarray(blk, np.int32)
            if not np.isin(bk, (0,) + CANDIDATE_BLOCKS).all():
                raise RuntimeError("invalid-granularity: a given block size must be 0 or one of "
                                   "16/32/64/128 (selector.hpp:12)")
            self.plan_blk.copy_(torch.as_tensor(bk))
            bb = np.zeros((self.lay.batch, self.heads))
            bud = np.asarray(budgets, dtype=object)
            for b in range(self.lay.batch):
                flat = []
                for g in range(self.lay.kv_heads):
                    gb = list(bud[b][g]) if len(np.shape(bud[b][g])) else []
                    flat.extend(gb + [0.0] * (self.lay.group_size - len(gb)))
                bb[b] = flat
            self.plan_budgets.copy_(torch.as_tensor(bb))
        a.plan_blk = self.plan_blk.data_ptr()
        a.plan_budgets = self.plan_budgets.data_ptr()
        a.plan_volume = self.plan_volume.data_ptr()
        a.plan_cand_volumes = self.plan_cand.data_ptr()
        a.plan_kblocks = self.plan_kblocks.data_ptr()
        a.sel_bits = self.sel_bits.data_ptr()
        a.sel_words = self.sel_words
        return a

    def _finish(self, a, host, out, lse):
        o = self.o if out is None else out
        ls = self.lse if lse is None else lse
        a.o = o.data_ptr()
        a.lse = ls.data_ptr()
        check(LIB.fx_decode_step(self.eng.ctx, C.byref(self.lay), C.byref(a)))
        if host:
            return o.cpu().numpy().copy(), ls.cpu().numpy().copy()
        return o, ls

    # -- synthetic workload (workload.cpp) --------------------------------------
    def generate(self, spec: dict, seeds=None, layers=None, steps: int = 0) -> dict:
        """generate(spec) (workload.cpp:154-308) into this cache: batch entry b is
        layer layers[b] of the workload seeded seeds[b] (default seed + b, layer 0).
        Returns device tensors anchor [B][H][D], step_q [steps][B][H][D],
        new_k / new_v [steps][B][Hkv][D] and host archetypes [B][H]."""
        lay = self.lay
        B, H, D, Hkv = lay.batch, self.heads, lay.head_dim, lay.kv_heads
        sp = N.WorkloadSpec.make(**spec)
        seeds = np.ascontiguousarray(seeds if seeds is not None else [sp.seed + b for b in range(B)],
                                     np.uint64)
        layers = np.ascontiguousarray(layers if layers is not None else [0] * B, np.int32)
        dev = self.eng.device
        out = dict(anchor=torch.empty((B, H, D), dtype=torch.float32, device=dev),
                   step_q=torch.empty((max(steps, 1), B, H, D), dtype=torch.float32, device=dev),
                   new_k=torch.empty((max(steps, 1), B, Hkv, D), dtype=torch.float32, device=dev),
                   new_v=torch.empty((max(steps, 1), B, Hkv, D), dtype=torch.float32, device=dev))
        arch = np.zeros((B, H), np.int32)
        check(LIB.fx_generate(self.eng.ctx, C.byref(sp), C.byref(lay), seeds.ctypes.data,
                              layers.ctypes.data, _ptr(self.k), _ptr(self.v), _ptr(out["anchor"]),
                              int(steps), _ptr(out["step_q"]), _ptr(out["new_k"]),
                              _ptr(out["new_v"]), arch.ctypes.data))
        out["archetypes"] = arch
        return out

    # -- FXT1 traces (workload.cpp:311-433) -------------------------------------
    @staticmethod
    def trace_info(path: str) -> "N.TraceInfo":
        info = N.TraceInfo()
        check(LIB.fx_trace_info_read(path.encode(), C.byref(info)))
        return info

    def load_trace(self, path: str, layer: int = 0, b: int = 0) -> dict:
        """import_trace of one layer into batch entry b; returns the device
        query / decoded-row arrays and the host archetypes of that layer."""
        info = self.trace_info(path)
        H, D, Hkv, S = info.heads, info.head_dim, info.heads // info.group_size, info.decode_steps
        dev = self.eng.device
        out = dict(anchor=torch.empty((H, D), dtype=torch.float32, device=dev),
                   step_q=torch.empty((max(S, 1), H, D), dtype=torch.float32, device=dev),
                   new_k=torch.empty((max(S, 1), Hkv, D), dtype=torch.float32, device=dev),
                   new_v=torch.empty((max(S, 1), Hkv, D), dtype=torch.float32, device=dev))
        arch = np.zeros(H, np.int32)
        check(LIB.fx_trace_load(self.eng.ctx, path.encode(), int(layer), C.byref(self.lay), int(b),
                                _ptr(self.k), _ptr(self.v), _ptr(out["anchor"]), _ptr(out["step_q"]),
                                _ptr(out["new_k"]), _ptr(out["new_v"]), arch.ctypes.data))
        out["archetypes"] = arch
        return out

    def save_trace(self, path: str, info: "N.TraceInfo", entries, anchor=None, step_q=None,
                   new_k=None, new_v=None, archetypes=None) -> None:
        """export_trace: trace layer ly = batch entry entries[ly]; per-layer
        device arrays anchor [layers][H][D], step_q [layers][steps][H][D],
        new_k / new_v [layers][steps][Hkv][D]; host archetypes [layers][H]."""
        ent = np.ascontiguousarray(entries, np.int32)
        arch = None if archetypes is None else np.ascontiguousarray(archetypes, np.int32)
        check(LIB.fx_trace_save(self.eng.ctx, path.encode(), C.byref(info), C.byref(self.lay),
                                ent.ctypes.data, _ptr(self.k), _ptr(self.v), _ptr(anchor),
                                _ptr(step_q), _ptr(new_k), _ptr(new_v),
                                None if arch is None else arch.ctypes.data, None, None))

    # -- output-aware labels (budget_oracle.cpp) --------------------------------
    def label_heads(self, q: torch.Tensor, tau: float = 0.10, output_only: bool = False) -> dict:
        """Oracle head properties of every query head (pipeline.cpp:256-276):
        o_full, the per-sequence normalizer, label_streaming, min_budget at blk
        1/16/32/64/128 and fit_curve -> dict of device tensors (bgt0, kslope,
        streaming [B][H]; budgets, blocks [B][H][5]; o_full [B][H][D] f64;
        normalizer [B]).  The metadata levels must have been built."""
        lay = self.lay
        B, H, D = lay.batch, self.heads, lay.head_dim
        dev = self.eng.device
        qd = q.to(dev, torch.float32).contiguous()
        out = dict(o_full=torch.empty((B, H, D), dtype=torch.float64, device=dev),
                   normalizer=torch.empty(B, dtype=torch.float64, device=dev),
                   budgets=torch.empty((B, H, 5), dtype=torch.float64, device=dev),
                   blocks=torch.empty((B, H, 5), dtype=torch.int64, device=dev),
                   bgt0=torch.empty((B, H), dtype=torch.float64, device=dev),
                   kslope=torch.empty((B, H), dtype=torch.float64, device=dev),
                   streaming=torch.empty((B, H), dtype=torch.int32, device=dev))
        meta = (C.c_void_p * 4)(*[m.data_ptr() for m in self.meta])
        check(LIB.fx_label_heads(self.eng.ctx, C.byref(lay), _ptr(self.k), _ptr(self.v),
                                 self.l_new, meta, _ptr(qd), float(tau), 1 if output_only else 0,
                                 *[_ptr(out[n]) for n in ("o_full", "normalizer", "budgets",
                                                          "blocks", "bgt0", "kslope",
                                                          "streaming")]))
        return out

    # -- predictor features (features.cpp) ---------------------------------------
    STATS_SCALARS = 32

    def prefill_stats(self, anchor: torch.Tensor, tau: float = 0.10, layer: int = 0) -> torch.Tensor:
        """prefill_stats (features.cpp:86-157) of every head on the prefill cache
        (no decoded rows): flat records [B][H][32 + 3 D] f64 on the device (layout
        in include/fluxattn_b200.h).  Budget features: min_budget of the anchor at
        blk 16..128 (pipeline.cpp:37-46)."""
        lay = self.lay
        rec = torch.zeros((lay.batch, self.heads, self.STATS_SCALARS + 3 * lay.head_dim),
                          dtype=torch.float64, device=self.eng.device)
        meta = (C.c_void_p * 4)(*[m.data_ptr() for m in self.meta])
        a = anchor.to(self.eng.device, torch.float32).contiguous()
        check(LIB.fx_prefill_stats(self.eng.ctx, C.byref(lay), _ptr(self.k), _ptr(self.v), meta,
                                   _ptr(a), float(tau), int(layer), _ptr(rec)))
        return rec

    def decode_features(self, q: torch.Tensor, rec: torch.Tensor,
                        out: torch.Tensor = None) -> torch.Tensor:
        """decode_features (features.cpp:172-224) of every head -> [B][H][41] f64."""
        lay = self.lay
        f = out if out is not None else torch.empty((lay.batch, self.heads, 41), dtype=torch.float64,
                                                    device=self.eng.device)
        qd = q.to(self.eng.device, torch.float32).contiguous()
        check(LIB.fx_decode_features(self.eng.ctx, C.byref(lay), _ptr(self.k), _ptr(self.v),
                                     self.l_new, _ptr(qd), _ptr(rec), _ptr(f)))
        return f

    def predict_props(self, q: torch.Tensor, rec: torch.Tensor, model: "Predictor",
                      features: torch.Tensor = None, z: torch.Tensor = None, append=None):
        """decode_features -> normalize -> predict for every head
        (features.cpp:162-233, predictor.cpp:161-185, pipeline.cpp:277-290) ->
        (bgt0, kslope, streaming) device tensors [B][H], the props of step().
        append=(k_new, v_new) [B][Hkv][D]: the previous token is appended first
        (append_new, pipeline.cpp:406-412) and seen by the features; the step
        that follows then takes no append."""
        lay = self.lay
        dev = self.eng.device
        shape = (lay.batch, self.heads)
        if not hasattr(self, "_pp") or self._pp[0].shape != shape:
            self._pp = (torch.empty(shape, dtype=torch.float64, device=dev),
                        torch.empty(shape, dtype=torch.float64, device=dev),
                        torch.empty(shape, dtype=torch.int32, device=dev))
        b0, ks, st = self._pp
        qd = q.to(dev, torch.float32).contiguous()
        ak = av = None
        if append is not None:
            if self.lay.l_sink + self.lay.l_cpu + self.lay.l_local + self.l_new + 1 > self.lay.l_cap:
                raise ValueError("bad-shape: decoded rows exceed l_cap")
            ak = append[0].to(dev, torch.float32).contiguous()
            av = append[1].to(dev, torch.float32).contiguous()
        check(LIB.fx_predict_props(self.eng.ctx, C.byref(lay), _ptr(self.k), _ptr(self.v), self.l_new,
                                   _ptr(ak), _ptr(av), _ptr(qd), _ptr(rec), model.h, _ptr(features),
                                   _ptr(z), _ptr(b0), _ptr(ks), _ptr(st)))
        if append is not None:
            self.l_new += 1
        return b0, ks, st

    def selected_blocks(self, b: int, h: int) -> np.ndarray:
        """Ids of the blocks head h of sequence b selected in the last step."""
        g = h // self.lay.group_size
        blk = int(self.plan_blk[b, g].item())
        if blk == 0:
            return np.zeros(0, np.int64)
        nblk = (self.lay.l_cpu + blk - 1) // blk
        w = self.sel_bits[b, h].cpu().numpy().view(np.uint32)
        bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:nblk]
        return np.nonzero(bits)[0]


class Predictor:
    """A 41->256->384->3 head-property predictor resident on the device
    (predictor.cpp:161-185); params as the oracle's make_model dict."""

    NAMES = ("w1", "b1", "w2", "b2", "w3", "b3", "mu", "sigma")

    def __init__(self, engine: Engine, params: dict):
        self.eng = engine
        self._host = [np.ascontiguousarray(params[n], np.float64) for n in self.NAMES]
        h = C.c_void_p()
        check(LIB.fx_model_create(engine.ctx, *[a.ctypes.data for a in self._host], C.byref(h)))
        self.h = h

    def __call__(self, feats: torch.Tensor, z: torch.Tensor = None):
        """features [..][41] f64 device -> (bgt0, kslope, streaming) shaped like
        feats[..., 0]; z (optional, [..][3] f64) receives the raw logits."""
        shape = feats.shape[:-1]
        n = int(np.prod(shape)) if len(shape) else 1
        dev = self.eng.device
        b0 = torch.empty(shape, dtype=torch.float64, device=dev)
        ks = torch.empty(shape, dtype=torch.float64, device=dev)
        st = torch.empty(shape, dtype=torch.int32, device=dev)
        check(LIB.fx_predict(self.eng.ctx, self.h, n, _ptr(feats.contiguous()), _ptr(b0), _ptr(ks),
                             _ptr(st), _ptr(z)))
        return b0, ks, st

    def close(self):
        if getattr(self, "h", None):
            LIB.fx_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
