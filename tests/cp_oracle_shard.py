"""TEST INFRASTRUCTURE: a CPU stand-in for context_parallel.CPShard built on the
C oracle (oracle/fx_oracle.c), so the torch.distributed orchestration of the
context-parallel step (cp_decode_step + TorchComm) can run under gloo on CPU.
The global selection here is an independent restatement -- a plain sort of
every gathered entry -- not the per-list rank search of fx_cp_select."""
import numpy as np
import torch

from paper_2605_07719_b200.context_parallel import shard_bounds

SIGN = np.uint64(0x8000000000000000)


def f64_key(s: np.ndarray) -> np.ndarray:
    """Order-preserving u64 image of f64 scores (fx_common.cuh f64_key)."""
    u = np.asarray(s, np.float64).view(np.uint64).copy()
    u[u == SIGN] = 0  # -0.0 == +0.0
    neg = (u & SIGN) != 0
    return np.where(neg, ~u, u | SIGN)


class OracleShard:
    def __init__(self, co, rank, ranks, K, V, l_sink, l_cpu, l_local, G):
        self.co, self.rank, self.ranks = co, rank, ranks
        self.off, self.rows = shard_bounds(l_cpu, ranks)[rank]
        self.K, self.V = K, V  # full single-device caches [B][Hkv][rows][D] f32 (host)
        self.l_sink, self.l_cpu, self.l_local = l_sink, l_cpu, l_local
        self.B, self.Hkv, self.D = K.shape[0], K.shape[1], K.shape[3]
        self.G = G
        self.n_heads = self.B * self.Hkv * G
        self.cap = (self.rows + 15) // 16

    def _chunk_rows(self):
        return self.l_sink + self.off, self.l_sink + self.off + self.rows

    def candidates(self, q: torch.Tensor, fixed):
        blk, bgt = fixed
        self.blk = blk
        self.k = self.co.blocks_for_budget(bgt, self.l_cpu, blk)
        a, e = self._chunk_rows()
        nh, cap = self.n_heads, self.cap
        keys = np.zeros((nh, cap), np.uint64)
        ids = np.full((nh, cap), 0xffffffff, np.uint32)
        kth = np.zeros(nh, np.uint64)
        qn = q.numpy()
        for b in range(self.B):
            for g in range(self.Hkv):
                mins, maxs = self.co.build_metadata(self.K[b, g, a:e], blk)
                for j in range(self.G):
                    hi = (b * self.Hkv + g) * self.G + j
                    s = self.co.block_scores(qn[b, g * self.G + j], mins, maxs)
                    order = np.lexsort((np.arange(len(s)), -s))[:min(self.k, len(s))]
                    n = len(order)
                    keys[hi, :n] = f64_key(s[order])
                    ids[hi, :n] = order + self.off // blk
                    if self.k > 0 and n >= self.k:
                        kth[hi] = keys[hi, self.k - 1]
        self.keys, self.ids = keys, ids
        self.kth = torch.from_numpy(kth.view(np.int64))
        return self.kth

    def threshold(self, kth_all: torch.Tensor) -> int:
        T = kth_all.numpy().view(np.uint64).max(axis=0)
        self.thresh = T
        lim = np.maximum(T, np.uint64(1))
        self.keep = (self.keys >= lim[:, None]).sum(axis=1)
        return int(self.keep.max()) if self.n_heads else 0

    def head_candidates(self, m: int):
        k = np.zeros((self.n_heads, m), np.uint64)
        i = np.full((self.n_heads, m), 0xffffffff, np.uint32)
        w = min(m, self.cap)
        k[:, :w], i[:, :w] = self.keys[:, :w], self.ids[:, :w]
        return torch.from_numpy(k.view(np.int64)), torch.from_numpy(i.view(np.int32))

    def select(self, gkeys: torch.Tensor, gids: torch.Tensor, m: int) -> None:
        gk = gkeys.numpy().view(np.uint64)  # [R][n][m]
        gi = gids.numpy().view(np.uint32)
        lo_id, hi_id = self.off // self.blk, (self.off + self.rows + self.blk - 1) // self.blk
        self.selected = {}
        for h in range(self.n_heads):
            lim = max(int(self.thresh[h]), 1)
            ent = [(int(gk[r, h, j]), int(gi[r, h, j])) for r in range(self.ranks) for j in range(m)
                   if int(gk[r, h, j]) >= lim]
            ent.sort(key=lambda x: (-x[0], x[1]))
            top = [i for _, i in ent[:self.k]]
            self.selected[h] = sorted(i for i in top if lo_id <= i < hi_id)

    def attend(self, q: torch.Tensor):
        qn = q.numpy()
        o = np.zeros((self.B, self.Hkv * self.G, self.D))
        lse = np.full((self.B, self.Hkv * self.G), -np.inf)
        a, _ = self._chunk_rows()
        for b in range(self.B):
            for g in range(self.Hkv):
                for j in range(self.G):
                    h = g * self.G + j
                    hi = (b * self.Hkv + g) * self.G + j
                    rows = []
                    if self.rank == 0:
                        rows += list(range(self.l_sink))
                    for blk_id in self.selected[hi]:
                        r0 = blk_id * self.blk - self.off
                        rows += [a + r for r in range(r0, min(r0 + self.blk, self.rows))]
                    if self.rank == self.ranks - 1:
                        t0 = self.l_sink + self.l_cpu
                        rows += list(range(t0, t0 + self.l_local))
                    if rows:
                        oh, lh, _ = self.co.gathered_attention(qn[b, h], self.K[b, g], self.V[b, g],
                                                               np.asarray(rows, np.uint32))
                        o[b, h], lse[b, h] = oh, lh
        return torch.from_numpy(o), torch.from_numpy(lse)

    def combine(self, o_all, lse_all, o, lse):
        oa, la = o_all.numpy(), lse_all.numpy()
        M = la.max(axis=0)
        w = np.where(np.isfinite(la), np.exp(la - M[None]), 0.0)
        den = w.sum(axis=0)
        o[...] = torch.from_numpy((w[..., None] * oa).sum(axis=0) / den[..., None])
        lse[...] = torch.from_numpy(M + np.log(den))
