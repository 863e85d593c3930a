"""Hybrid HBM / host-memory KV for the batched decode step -- SURVEY §8f-4 on a
B200.

The reference's hybrid execution (scheduler.cpp:129-279; scheduler.hpp:48-68)
keeps part of the KV in host memory and lets host workers take the
low-priority tasks -- the ones with the smallest selection volume V (Eq. 3,
selector.cpp:9-13) -- from the same V-ordered queue the accelerator drains
from the top (enqueue_batch, scheduler.cpp:65-76).  On a B200 the arithmetic
stays on the GPU; what moves to the host is the *data*: a host-tier
sequence's K/V lives in pinned host memory that the same kernels read
through the unified address space (TMA tensor maps and bulk copies work on
mapped host memory, over PCIe / NVLink-C2C), while its block metadata stays in
HBM.  Only the metadata scan runs at HBM speed for it; the selected blocks and
the default rows (a few per cent of the context) cross the link.  So the
queue's order decides residency instead of who computes:

  * assign_tiers: sequences by their summed group volume V, the largest in HBM
    (they move the most bytes), the smallest in host memory -- the tail of the
    reference's priority order, which its host workers would take;
  * step: the HBM tier and the host tier run as two concurrent decode steps on
    two streams (each its own C-ABI context), the host tier's link-bound
    attention overlapping the HBM tier's; outputs land in one [B][H][D] array.

Selections are identical to a single all-HBM step over the same data (same
kernels, same plan), outputs equal up to the split-K partition of the smaller
launches (which sets where the softmax partials and their bf16 P tiles are
cut; within the bf16 bar, tests/test_tiered.py).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from .fluxattn import Engine, SparseDecoder


def assign_tiers(volumes: Sequence[float], hbm_sequences: int) -> list:
    """Host-tier sequence ids: all but the `hbm_sequences` largest volumes
    (ties: the lower id stays in HBM, as enqueue_batch breaks ties)."""
    v = np.asarray(volumes, np.float64)
    order = sorted(range(len(v)), key=lambda b: (-v[b], b))  # priority order
    return sorted(order[hbm_sequences:])


def sequence_volumes(engine: Engine, props, l_cpu: int, group_size: int) -> np.ndarray:
    """Summed plan_group volume of every sequence (Eq. 3 over its groups),
    planned on the device from head properties (bgt0, kslope, streaming) [B][H]."""
    from .fluxattn import HeadProperties
    b0, ks, st = (np.asarray(t.cpu() if isinstance(t, torch.Tensor) else t) for t in props)
    B, H = b0.shape
    groups = [[HeadProperties(float(b0[b, h]), float(ks[b, h]), bool(st[b, h]))
               for h in range(g * group_size, (g + 1) * group_size)]
              for b in range(B) for g in range(H // group_size)]
    plans = engine.plan_groups(groups, l_cpu)
    vol = np.array([p.volume for p in plans]).reshape(B, H // group_size)
    return vol.sum(1)


class TieredDecoder:
    """A batch split into an HBM tier and a host-memory tier (pinned K/V)."""

    def __init__(self, engine: Engine, batch: int, kv_heads: int, group_size: int, head_dim: int,
                 l_sink: int, l_cpu: int, l_local: int, host_sequences: Sequence[int], max_new: int = 64,
                 dtype: str = "bf16"):
        self.batch = batch
        self.host_ids = sorted(set(int(b) for b in host_sequences))
        if any(b < 0 or b >= batch for b in self.host_ids):
            raise RuntimeError("bad-shape: host sequence id outside the batch")
        self.dev_ids = [b for b in range(batch) if b not in self.host_ids]
        self.heads = kv_heads * group_size
        self.head_dim = head_dim
        dev = engine.device
        self.eng = engine
        self.streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        self.engines = (engine, Engine(dev.index))  # one context per tier: concurrent steps
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        cap = SparseDecoder.cap_rows(l_sink + l_cpu + l_local, max_new)
        self.tiers = []
        for t, ids in enumerate((self.dev_ids, self.host_ids)):
            if not ids:
                self.tiers.append(None)
                continue
            kv = {}
            if t == 1:  # pinned host memory, addressed by the kernels through UVA
                shape = (len(ids), kv_heads, cap, head_dim)
                kv = dict(k=torch.zeros(shape, dtype=tdt).pin_memory(),
                          v=torch.zeros(shape, dtype=tdt).pin_memory())
            self.tiers.append(SparseDecoder(self.engines[t], len(ids), kv_heads, group_size, head_dim,
                                            l_sink, l_cpu, l_local, max_new=max_new, dtype=dtype, **kv))
        self._slot = {b: (0, i) for i, b in enumerate(self.dev_ids)}
        self._slot.update({b: (1, i) for i, b in enumerate(self.host_ids)})
        self._idx = [torch.as_tensor(ids, dtype=torch.long, device=dev) if ids else None
                     for ids in (self.dev_ids, self.host_ids)]

    # -- data ----------------------------------------------------------------
    def load_group(self, b: int, g: int, k: np.ndarray, v: np.ndarray) -> None:
        t, i = self._slot[b]
        self.tiers[t].load_group(i, g, k, v)

    def build_metadata(self) -> None:
        """K1 for both tiers (the host tier's K streams over the link once)."""
        for dec in self.tiers:
            if dec is not None:
                dec.eng.sync_stream()
                dec.build_metadata()

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor) -> None:
        """append_new for every sequence: [B][Hkv][D] f32 device rows."""
        for t, dec in enumerate(self.tiers):
            if dec is not None:
                dec.eng.sync_stream()
                dec.append(k_new.index_select(0, self._idx[t]), v_new.index_select(0, self._idx[t]))

    @property
    def l_new(self) -> int:
        return next(d.l_new for d in self.tiers if d is not None)

    # -- one decode step --------------------------------------------------------
    def step(self, q: torch.Tensor, props=None, fixed=None, out: Optional[torch.Tensor] = None,
             lse: Optional[torch.Tensor] = None):
        """q [B][H][D] f32 device; props = (bgt0, kslope, streaming) [B][H] device
        tensors or fixed = (blk, bgt).  Both tiers step concurrently."""
        cur = torch.cuda.current_stream(self.eng.device)
        o = out if out is not None else torch.empty((self.batch, self.heads, self.head_dim),
                                                   dtype=torch.float32, device=q.device)
        ls = lse if lse is not None else torch.empty((self.batch, self.heads), dtype=torch.float32,
                                                    device=q.device)
        parts = []
        for t, dec in enumerate(self.tiers):
            if dec is None:
                continue
            s = self.streams[t]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                dec.eng.sync_stream()
                idx = self._idx[t]
                kw = dict(fixed=fixed) if fixed is not None else \
                    dict(props=tuple(p.index_select(0, idx) for p in props))
                ot, lt = dec.step(q.index_select(0, idx), **kw)
                parts.append((t, ot, lt))
        for t, ot, lt in parts:
            cur.wait_stream(self.streams[t])
            o.index_copy_(0, self._idx[t], ot)
            ls.index_copy_(0, self._idx[t], lt)
        self.eng.sync_stream()
        return o, ls

    def selected_blocks(self, b: int, h: int) -> np.ndarray:
        t, i = self._slot[b]
        return self.tiers[t].selected_blocks(i, h)
