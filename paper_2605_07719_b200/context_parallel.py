"""Context-parallel sparse decode over cpu-segment shards (config C5: 1M-token
context, batch 4, 8 x B200).

The reference is single-device: ``execute_task``
(scheduler.cpp:78-96) runs topk_blocks (block_index.cpp:55-83) over the whole
cpu segment and merge_into (attention.cpp:89-104) over the partials.  Here the
cpu segment of every (b, g) is split into contiguous 128-row-aligned shards,
one per rank, with the sink rows on rank 0 and local + decoded rows on the last
rank.  A block of any candidate granularity (16..128) then lives whole on one
shard and keeps its global id, and one decode step is

    1. fx_cp_candidates  plan (whole-sequence L_cpu), local top-min(k, nblk)
                          with exact reference scores, sorted
    2. all-gather kth  -> fx_cp_threshold   T = max_r (local k-th key)
    3. all-gather the entries with key >= T -> fx_cp_select   global ranks
    4. fx_decode_step  (given plan + given selection) -> shard (o, lse)
    5. all-gather (o, lse) -> fx_cp_combine (LSE merge)

which reproduces the single-device selection bit-exactly (argument in
csrc/fx_cp.cu) and its output within the f32 merge tolerance.  All three
exchanges are small (B*H*8 B, ~B*H*k*12 B, B*H*(D+1)*4 B); they go through
``torch.distributed`` (NCCL over NVLink on the box).  ``LoopbackComm`` runs all
shards of a step in one process (tests, and the single-GPU measurement), with
the identical phase code.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np
import torch

from . import _native as N
from ._native import LIB, check
from .fluxattn import Engine, SparseDecoder

ALIGN = 128  # shard boundaries: multiple of every candidate granularity


def shard_bounds(l_cpu: int, ranks: int) -> List[Tuple[int, int]]:
    """(offset, rows) of each rank's cpu chunk: equal 128-aligned chunks, the
    last one holding the remainder (possibly empty chunks at the end)."""
    chunk = -(-l_cpu // ranks)
    chunk = -(-chunk // ALIGN) * ALIGN
    out = []
    for r in range(ranks):
        a = min(l_cpu, r * chunk)
        out.append((a, min(l_cpu, a + chunk) - a))
    return out


def shard_kv(k_full: torch.Tensor, l_sink: int, l_cpu: int, l_local: int, rank: int, ranks: int,
             max_new: int = 64) -> torch.Tensor:
    """Rank `rank`'s rows of a single-device cache [B][Hkv][rows][D] (sink | cpu |
    local ...), laid out as that shard's SparseDecoder cache."""
    off, n = shard_bounds(l_cpu, ranks)[rank]
    last = rank == ranks - 1
    parts = []
    if rank == 0:
        parts.append(k_full[:, :, :l_sink])
    parts.append(k_full[:, :, l_sink + off:l_sink + off + n])
    if last:
        parts.append(k_full[:, :, l_sink + l_cpu:l_sink + l_cpu + l_local])
    rows = sum(p.shape[2] for p in parts)
    cap = SparseDecoder.cap_rows(rows, max_new if last else 0)
    out = torch.zeros(k_full.shape[:2] + (cap, k_full.shape[3]), dtype=k_full.dtype,
                      device=k_full.device)
    out[:, :, :rows] = torch.cat(parts, dim=2)
    return out


class TorchComm:
    """Exchanges of one rank over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.ranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, local: Sequence[torch.Tensor]) -> torch.Tensor:
        (t,) = local
        t = t.contiguous().reshape(1, -1)
        out = torch.empty((self.ranks, t.shape[1]), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.view((self.ranks,) + tuple(local[0].shape))

    def max_int(self, local: Sequence[int], device) -> int:
        (v,) = local
        t = torch.tensor([int(v)], dtype=torch.int64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())


class LoopbackComm:
    """All ranks' shards in this process: the exchanges are stacks."""

    def __init__(self, ranks: int):
        self.ranks = ranks

    def all_gather(self, local: Sequence[torch.Tensor]) -> torch.Tensor:
        assert len(local) == self.ranks
        return torch.stack([t.contiguous() for t in local])

    def max_int(self, local: Sequence[int], device) -> int:
        return max(int(v) for v in local)


class CPShard:
    """One rank's share of a context-parallel batch: a SparseDecoder over its
    cpu chunk (+ sink rows on rank 0, + local and decoded rows on the last)."""

    def __init__(self, engine: Engine, rank: int, ranks: int, batch: int, kv_heads: int,
                 group_size: int, head_dim: int, l_sink: int, l_cpu_total: int, l_local: int,
                 max_new: int = 64, dtype: str = "bf16", k: torch.Tensor = None,
                 v: torch.Tensor = None):
        self.rank, self.ranks = rank, ranks
        off, n = shard_bounds(l_cpu_total, ranks)[rank]
        if n == 0:
            raise RuntimeError("empty-context: more shards than 128-row cpu chunks")
        last = rank == ranks - 1
        self.dec = SparseDecoder(engine, batch, kv_heads, group_size, head_dim,
                                 l_sink if rank == 0 else 0, n, l_local if last else 0,
                                 max_new if last else 0, dtype, k, v)
        self.dec.l_cpu_total = l_cpu_total
        self.dec.cpu_offset = off
        self.eng = engine
        self.offset, self.rows = off, n
        nh = batch * kv_heads * group_size
        self.n_heads = nh
        self.cap = (n + 15) // 16
        dev = engine.device
        self.keys = torch.zeros((nh, self.cap), dtype=torch.int64, device=dev)  # u64 keys
        self.ids = torch.zeros((nh, self.cap), dtype=torch.int32, device=dev)
        self.count = torch.zeros(nh, dtype=torch.int32, device=dev)
        self.kth = torch.zeros(nh, dtype=torch.int64, device=dev)
        self.thresh = torch.zeros(nh, dtype=torch.int64, device=dev)
        self.keep = torch.zeros(nh, dtype=torch.int32, device=dev)
        self.sel = torch.zeros((batch, kv_heads * group_size, self.dec.sel_words), dtype=torch.int32,
                               device=dev)
        self.o = torch.empty((batch, kv_heads * group_size, head_dim), dtype=torch.float32, device=dev)
        self.lse = torch.empty((batch, kv_heads * group_size), dtype=torch.float32, device=dev)

    @property
    def is_last(self) -> bool:
        return self.rank == self.ranks - 1

    # -- phases ------------------------------------------------------------------
    def candidates(self, q: torch.Tensor, **plan) -> torch.Tensor:
        d = self.dec
        a = d._args(q, plan.get("props"), plan.get("fixed"), plan.get("full", False),
                    plan.get("blk"), plan.get("budgets"))
        check(LIB.fx_cp_candidates(self.eng.ctx, C.byref(d.lay), C.byref(a), self.cap,
                                   self.keys.data_ptr(), self.ids.data_ptr(),
                                   self.count.data_ptr(), self.kth.data_ptr()))
        return self.kth

    def threshold(self, kth_all: torch.Tensor) -> int:
        check(LIB.fx_cp_threshold(self.eng.ctx, self.ranks, self.n_heads, self.cap,
                                  self.keys.data_ptr(), kth_all.data_ptr(),
                                  self.thresh.data_ptr(), self.keep.data_ptr()))
        return int(self.keep.max().item()) if self.n_heads else 0

    def head_candidates(self, m: int) -> Tuple[torch.Tensor, torch.Tensor]:
        """This shard's first m sorted entries per head (the exchanged slice)."""
        if m <= self.cap:
            return self.keys[:, :m], self.ids[:, :m]
        pad = m - self.cap
        return (torch.nn.functional.pad(self.keys, (0, pad)),
                torch.nn.functional.pad(self.ids, (0, pad), value=-1))

    def select(self, gkeys: torch.Tensor, gids: torch.Tensor, m: int) -> None:
        d = self.dec
        check(LIB.fx_cp_select(self.eng.ctx, C.byref(d.lay), self.ranks, self.rank, m,
                               gkeys.data_ptr(), gids.data_ptr(), self.thresh.data_ptr(),
                               d.plan_kblocks.data_ptr(), d.plan_blk.data_ptr(), self.offset,
                               self.sel.data_ptr(), d.sel_words))

    def attend(self, q: torch.Tensor):
        return self.dec.step(q, blk="keep", out=self.o, lse=self.lse, sel_in=self.sel)

    def combine(self, o_all: torch.Tensor, lse_all: torch.Tensor, o: torch.Tensor,
                lse: torch.Tensor) -> None:
        D = o.shape[-1]
        check(LIB.fx_cp_combine(self.eng.ctx, self.ranks, self.n_heads, D, o_all.data_ptr(),
                                lse_all.data_ptr(), o.data_ptr(), lse.data_ptr()))

    def global_selection(self, b: int, h: int) -> torch.Tensor:
        """Global ids of the blocks this shard selected for head h of b."""
        g = h // self.dec.lay.group_size
        blk = int(self.dec.plan_blk[b, g].item())
        if blk == 0:
            return np.zeros(0, np.int64)
        words = self.sel[b, h].cpu().numpy().view(np.uint32)
        nblk = (self.rows + blk - 1) // blk
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:nblk]
        return np.nonzero(bits)[0] + self.offset // blk


def cp_decode_step(shards: Sequence, comm, q: torch.Tensor, out: Sequence[Tuple[torch.Tensor, torch.Tensor]] = None,
                   **plan):
    """One context-parallel decode step over this process's shards (one per
    rank under torch.distributed, all of them under LoopbackComm).  Returns the
    merged (o [B][H][D], lse [B][H]) of each local shard (identical on every
    rank)."""
    for s in shards:
        s.candidates(q, **plan)
    kth_all = comm.all_gather([s.kth for s in shards])
    m = comm.max_int([s.threshold(kth_all) for s in shards], q.device)
    m = max(m, 1)
    cand = [s.head_candidates(m) for s in shards]
    gkeys = comm.all_gather([c[0] for c in cand])
    gids = comm.all_gather([c[1] for c in cand])
    for s in shards:
        s.select(gkeys, gids, m)
    parts = [s.attend(q) for s in shards]
    o_all = comm.all_gather([p[0] for p in parts])
    lse_all = comm.all_gather([p[1] for p in parts])
    res = []
    for i, s in enumerate(shards):
        if out is not None:
            o, lse = out[i]
        else:
            o, lse = torch.empty_like(s.o), torch.empty_like(s.lse)
        s.combine(o_all, lse_all, o, lse)
        res.append((o, lse))
    return res


# ---------------------------------------------------------------------------
# one-shot exchanges over peer memory (no NCCL): fx_cp_select_peer /
# fx_cp_combine_peer read the other ranks' candidate lists and (o, lse)
# partials where they live, after each rank's ready flag
# ---------------------------------------------------------------------------
DIST_BINS = 2048  # fx_cp.cu kDBins


class PeerShard(CPShard):
    """A CPShard whose exchange tables (candidates, k-th keys, partials, ready
    flags) are double-buffered by step parity and exported to the peers.  Two
    sets suffice: a rank's step s+1 select waits for every peer's step s+1
    candidates, which each peer publishes only after its step s combine has
    read this rank's set s."""

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        dev = self.eng.device
        nh, D = self.n_heads, self.dec.lay.head_dim
        B, H = self.dec.lay.batch, self.dec.heads
        self.sets = []
        for _ in range(2):
            self.sets.append(dict(
                keys=torch.zeros((nh, self.cap), dtype=torch.int64, device=dev),
                ids=torch.zeros((nh, self.cap), dtype=torch.int32, device=dev),
                count=torch.zeros(nh, dtype=torch.int32, device=dev),
                kth=torch.zeros(nh, dtype=torch.int64, device=dev),
                o=torch.zeros((B, H, D), dtype=torch.float32, device=dev),
                lse=torch.zeros((B, H), dtype=torch.float32, device=dev),
                stats=torch.zeros((nh, 4), dtype=torch.float64, device=dev),
                hist=torch.zeros((nh, DIST_BINS), dtype=torch.int32, device=dev),
                defc=torch.zeros((nh, 2), dtype=torch.int32, device=dev)))
        # [parity][slot]: 0 candidates / stats, 1 histograms, 2 bands, 3 partials
        self.flags = torch.zeros((2, 4), dtype=torch.int64, device=dev)
        self.approx = None  # [nh][cap] f32, the bracket protocol's local scores

    def table(self, parity: int) -> "N.CpPeer":
        st = self.sets[parity]
        return N.CpPeer(st["keys"].data_ptr(), st["ids"].data_ptr(), st["kth"].data_ptr(),
                        st["o"].data_ptr(), st["lse"].data_ptr(), self.flags[parity].data_ptr(),
                        self.cap, st["stats"].data_ptr(), st["hist"].data_ptr(), st["defc"].data_ptr())

    def exported(self):
        """(name, handle bytes, offset) of every exchange buffer, for the peers."""
        out = []
        bufs = [(f"{n}{p}", self.sets[p][n]) for p in range(2)
                for n in ("keys", "ids", "kth", "o", "lse", "stats", "hist", "defc")] + [("flags", self.flags)]
        for name, t in bufs:
            h = C.create_string_buffer(64)
            off = C.c_int64(0)
            check(LIB.fx_ipc_handle(C.c_void_p(t.data_ptr()), h, C.byref(off)))
            out.append((name, h.raw, off.value))
        return out

    def dist_phase(self, q, parity, phase, tables: "PeerTables", peers, stamp, **plan):
        """One phase of the distributed bracket selection (fx_cp_dist_phase)."""
        d = self.dec
        if phase == 0:
            a = d._args(q, plan.get("props"), plan.get("fixed"), plan.get("full", False),
                        plan.get("blk"), plan.get("budgets"))
            if self.approx is None:
                self.approx = torch.empty((self.n_heads, self.cap), dtype=torch.float32,
                                          device=self.eng.device)
        else:
            a = d.args
        a.sel_bits = self.sel.data_ptr()
        a.sel_words = d.sel_words
        check(LIB.fx_cp_dist_phase(self.eng.ctx, C.byref(d.lay), C.byref(a), phase, tables.ranks,
                                   self.rank, peers, stamp, self.approx.data_ptr(), self.cap))
        if phase < 3:
            check(LIB.fx_cp_signal(self.eng.ctx, C.c_void_p(self.flags[parity].data_ptr()), phase, stamp))

    def candidates_into(self, q, parity, **plan):
        st = self.sets[parity]
        d = self.dec
        a = d._args(q, plan.get("props"), plan.get("fixed"), plan.get("full", False),
                    plan.get("blk"), plan.get("budgets"))
        check(LIB.fx_cp_candidates(self.eng.ctx, C.byref(d.lay), C.byref(a), self.cap,
                                   st["keys"].data_ptr(), st["ids"].data_ptr(),
                                   st["count"].data_ptr(), st["kth"].data_ptr()))


class PeerTables:
    """The R ranks' exchange tables as device pointers of this process: local
    shards directly, remote ranks through CUDA IPC (opened once)."""

    def __init__(self, engine: Engine, ranks: int):
        self.eng = engine
        self.ranks = ranks
        self.tabs = [[None] * ranks for _ in range(2)]  # [parity][rank] -> CpPeer
        self._opened = []

    def add_local(self, shard: PeerShard) -> None:
        for p in range(2):
            self.tabs[p][shard.rank] = shard.table(p)

    def add_remote(self, rank: int, cap: int, exported) -> None:
        ptr = {}
        for name, handle, off in exported:
            d = C.c_void_p()
            check(LIB.fx_ipc_open(self.eng.ctx, handle, C.byref(d)))
            self._opened.append(d)
            ptr[name] = d.value + off
        for p in range(2):
            self.tabs[p][rank] = N.CpPeer(ptr[f"keys{p}"], ptr[f"ids{p}"], ptr[f"kth{p}"],
                                          ptr[f"o{p}"], ptr[f"lse{p}"], ptr["flags"] + p * 32, cap,
                                          ptr[f"stats{p}"], ptr[f"hist{p}"], ptr[f"defc{p}"])

    def array(self, parity: int):
        arr = (N.CpPeer * self.ranks)(*self.tabs[parity])
        return arr

    def close(self) -> None:
        for d in self._opened:
            LIB.fx_ipc_close(self.eng.ctx, d)
        self._opened = []

    @classmethod
    def over_dist(cls, engine: Engine, shard: PeerShard, group=None) -> "PeerTables":
        """Exchange IPC handles of every rank's tables over torch.distributed."""
        import torch.distributed as dist
        R = dist.get_world_size(group)
        mine = (shard.rank, shard.cap, shard.exported())
        allx = [None] * R
        dist.all_gather_object(allx, mine, group=group)
        t = cls(engine, R)
        t.add_local(shard)
        for rank, cap, exported in allx:
            if rank != shard.rank:
                t.add_remote(rank, cap, exported)
        return t


def cp_decode_step_peer(shards: Sequence[PeerShard], tables: PeerTables, q: torch.Tensor,
                        stamp: int, out: Sequence[Tuple[torch.Tensor, torch.Tensor]] = None, **plan):
    """One context-parallel decode step with the one-shot peer exchanges.
    `stamp` increases by one per step (>= 1); this process's shards run in
    order on one stream (all shards in one process, or one per rank)."""
    par = stamp % 2
    peers = tables.array(par)
    for s in shards:
        s.candidates_into(q, par, **plan)
        check(LIB.fx_cp_signal(s.eng.ctx, C.c_void_p(s.flags[par].data_ptr()), 0, stamp))
    for s in shards:
        d = s.dec
        check(LIB.fx_cp_select_peer(s.eng.ctx, C.byref(d.lay), tables.ranks, s.rank, peers, stamp,
                                    d.plan_kblocks.data_ptr(), d.plan_blk.data_ptr(), s.offset,
                                    s.sel.data_ptr(), d.sel_words))
    for s in shards:
        st = s.sets[par]
        s.dec.step(q, blk="keep", out=st["o"], lse=st["lse"], sel_in=s.sel)
        check(LIB.fx_cp_signal(s.eng.ctx, C.c_void_p(s.flags[par].data_ptr()), 3, stamp))
    res = []
    for i, s in enumerate(shards):
        if out is not None:
            o, lse = out[i]
        else:
            o, lse = torch.empty_like(s.o), torch.empty_like(s.lse)
        D = o.shape[-1]
        check(LIB.fx_cp_combine_peer(s.eng.ctx, tables.ranks, s.n_heads, D, peers, stamp,
                                     o.data_ptr(), lse.data_ptr()))
        res.append((o, lse))
    return res


def cp_decode_step_dist(shards: Sequence[PeerShard], tables: PeerTables, q: torch.Tensor,
                        stamp: int, out: Sequence[Tuple[torch.Tensor, torch.Tensor]] = None, **plan):
    """cp_decode_step_peer with the selection distributed as the single-device
    bracket (fx_cp_dist_phase): the ranks exchange per-head score ranges,
    2048-bin histograms and the exact-scored band around the global k-th
    score, so only the band is ever exact-scored or sorted.  Same selection
    as the one-device step, bit for bit."""
    par = stamp % 2
    peers = tables.array(par)
    for phase in range(4):
        for s in shards:
            s.dist_phase(q, par, phase, tables, peers, stamp, **plan)
    res = []
    for s in shards:
        st = s.sets[par]
        s.dec.step(q, blk="keep", out=st["o"], lse=st["lse"], sel_in=s.sel)
        check(LIB.fx_cp_signal(s.eng.ctx, C.c_void_p(s.flags[par].data_ptr()), 3, stamp))
    for i, s in enumerate(shards):
        if out is not None:
            o, lse = out[i]
        else:
            o, lse = torch.empty_like(s.o), torch.empty_like(s.lse)
        check(LIB.fx_cp_combine_peer(s.eng.ctx, tables.ranks, s.n_heads, o.shape[-1], peers, stamp,
                                     o.data_ptr(), lse.data_ptr()))
        res.append((o, lse))
    return res
