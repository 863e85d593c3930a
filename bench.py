#!/usr/bin/env python
"""Fluxion sparse-attention decode step on B200 -- the BASELINE.json metric.

Workload (BASELINE.json configs[1], "C2"): one Llama-3-8B-shaped decode layer
(32 query / 8 KV heads, head_dim 128), 131072-token context per sequence
(sink 64 | cpu 130752 | local 256 | decoded rows), batch 16 per GPU, bf16 KV,
synthetic N(0,1) K/V generated on device.  Budgets: per-head properties
(bgt0 ~ U(0.01, 0.05), k ~ U(0, 0.01), streaming ~ Bernoulli(0.5), seed 1;
SURVEY §8d perf run) -> on-device plan_group picks each group's granularity
(16/32/64/128) and per-head budgets every step.

One timed step = K5 plan -> K2 score/select (+ fused worklist) -> K3/K4 sparse
GQA attention + fused LSE merge for all 512 heads of the batch, plus the append
of the step's new K/V row of every group.  Per-step working set is > 1 GB, far
above the 126 MB L2, so no flush is needed between steps.

Multi-GPU (torchrun): weak scaling, every rank decodes its own batch of 16
(batch x KV-head sharding needs no collective); value = aggregate steps/s.

--impl reference: the reference's own executed CPU path (oracle/_ref, the
unmodified sources compiled here) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-attn decode steps/s at 128K ctx, bs=16; achieved HBM GB/s vs peak"
UNIT = "steps/s"
H, HKV, G, D = 32, 8, 4, 128
L_SINK, L_LOCAL = 64, 256


def args_parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--context", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quick", action="store_true", help="profiling run: timed loop only")
    ap.add_argument("--data", default="reference", choices=["reference", "normal"],
                    help="reference: the reference generator's workload (generate(spec), on "
                         "device); normal: plain N(0,1) K/V")
    ap.add_argument("--cp-exchange", default="dist", choices=["dist", "peer", "collective"],
                    help="c5 exchanges: peer-memory one-shot kernels, or torch.distributed "
                         "all-gathers (NCCL)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4", "c5"],
                    help="c2: one layer, batch 16 (the metric's config); c4: 32 layers x batch 8 "
                         "per GPU (configs[3], one 8-GPU shard), the layers' independent tasks "
                         "batched into one step like run_decode's single queue (pipeline.cpp:354); "
                         "c5: 1M context, batch 4, context-parallel over the torchrun ranks "
                         "(configs[4]; one rank = the single-device step)")
    a = ap.parse_args()
    if a.workload == "c4":
        a.layers, a.seqs = 32, 8
        a.batch = a.layers * a.seqs  # (layer, sequence) pairs: independent (b, g) tasks
    else:
        a.layers, a.seqs = 1, a.batch
    return a


def head_props(batch, seed=1):
    rng = np.random.default_rng(seed)
    bgt0 = rng.uniform(0.01, 0.05, (batch, H))
    kslope = rng.uniform(0.0, 0.01, (batch, H))
    streaming = (rng.random((batch, H)) < 0.5).astype(np.int32)
    return bgt0, kslope, streaming


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel, workload="c2"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the
    committed `ncu --set full` extract of the same bench command and workload
    (profiles/ncu_traffic.json for c2, profiles/ncu_traffic_<workload>.json
    otherwise; written by profiles/summarize_ncu.py); None if absent."""
    name = "ncu_traffic.json" if workload == "c2" else f"ncu_traffic_{workload}.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            t = json.load(f)
        for name, rec in t["kernels"].items():
            if kernel in name:
                return rec
    except Exception:
        pass
    return None


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 5 ms on a
    side thread during the timed region (plus one sample at each end); the
    samples also go to gpurun_out/clocks_rank<i>.csv."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")
        self.rows = []
        self.h = None
        self.thread = None

    def _sample(self):
        import pynvml as nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except AttributeError:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((time.time(), sm, mx, r))

    def start(self):
        import threading
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            try:  # the NVML device whose PCI bus id matches this CUDA device
                want = str(torch.cuda.get_device_properties(self.index).pci_bus_id).lower()[-7:]
                for i in range(nv.nvmlDeviceGetCount()):
                    h = nv.nvmlDeviceGetHandleByIndex(i)
                    bid = nv.nvmlDeviceGetPciInfo(h).busId
                    bid = (bid.decode() if isinstance(bid, bytes) else str(bid)).lower()
                    if bid.endswith(want):
                        self.h = h
                        break
            except Exception:
                pass
            self._sample()
        except Exception:
            self.h = None
            return
        self.stop_ev = threading.Event()

        def loop():
            while not self.stop_ev.wait(0.005):
                try:
                    self._sample()
                except Exception:
                    return
        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["unsampled"]}
        self._sample()
        self.stop_ev.set()
        self.thread.join()
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        with open(self.path, "w") as f:
            f.write("time,clocks.sm,clocks.max.sm,clocks_event_reasons\n")
            for t, sm, mx, r in self.rows:
                f.write(f"{t:.4f},{sm},{mx},{r:#x}\n")
        sm = [r[1] for r in self.rows]
        mx = [r[2] for r in self.rows]
        reasons = sorted({n for *_, r in self.rows for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "samples": len(sm), "reasons": reasons}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref) on a bounded sample
# ---------------------------------------------------------------------------
def reference_sample(ref, kv_groups, plans, queries, host_workers, repeats):
    """Run the reference's executed scheduler over one sequence's groups.

    kv_groups[g] = (K, V) position-ordered f32; plans[g] = (blk, budgets) or
    None for a streaming group (no task, like pipeline.cpp:334-337)."""
    batch = ref.batch()
    l_cpu = kv_groups[0][0].shape[0] - L_SINK - L_LOCAL
    n_tasks = 0
    for g, (k, v) in enumerate(kv_groups):
        if plans[g] is None:
            continue
        blk, budgets = plans[g]
        batch.add(k, v, (L_SINK, l_cpu, L_LOCAL, 0), queries[g * G:(g + 1) * G], blk, budgets)
        n_tasks += 1
    times = []
    for _ in range(repeats):
        sec, _ = batch.run(host_workers)
        times.append(sec)
    return times, n_tasks


def run_reference_arm(a):
    """--impl reference: the reference CPU path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import RefOracle
    ref = RefOracle()
    cores = os.cpu_count() or 1
    workers = max(1, cores - 1)
    l_cpu = a.context - L_SINK - L_LOCAL
    rng = np.random.default_rng(7)
    groups = []
    if a.data == "reference":  # the reference's own generator, sequence 0 (seed 1), layer 0
        w = ref.generate(seed=1, layers=1, heads=H, group_size=G, head_dim=D,
                         context_len=a.context, decode_steps=1)
        groups = [w.group_kv(0, g) for g in range(HKV)]
        q = w.queries(0, 0)
    else:
        for g in range(HKV):
            k = rng.standard_normal((a.context, D), dtype=np.float32)
            v = rng.standard_normal((a.context, D), dtype=np.float32)
            groups.append((k, v))
        q = rng.standard_normal((H, D)).astype(np.float32)
        q *= np.sqrt(D) / np.linalg.norm(q, axis=-1, keepdims=True)
    bgt0, ks, st = head_props(a.batch)
    plans = []
    for g in range(HKV):
        sl = slice(g * G, (g + 1) * G)
        p = ref.plan_group(bgt0[0, sl], ks[0, sl], st[0, sl], l_cpu)
        plans.append(None if p["streaming_group"] else (p["block_size"], p["budgets"]))
    times, n_tasks = reference_sample(ref, groups, plans, q, workers, a.warmup + a.steps)
    t = float(np.mean(times[a.warmup:])) if len(times) > a.warmup else float(np.mean(times))
    per_step = t * a.batch  # one sequence sampled; the batch has `batch` of them
    value = 1.0 / per_step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic: the reference's generate(spec), seed 1" if a.data == "reference"
                 else "synthetic N(0,1)"),
        "config": {"workload": "C2: Llama-3-8B layer (32q/8kv, d128), 128K ctx, batch 16, "
                               "per-head budgets + per-group granularity via plan_group",
                   "context": a.context, "global_batch": a.batch * a.gpus,
                   "sample": "1 of 16 sequences (8 KV groups) per step, extrapolated x16"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers + 1, "kind": "reference",
                         "sample": f"{n_tasks} retrieval-group tasks of 1 sequence per step, "
                                   f"run(queue, profile, RunMode::Executed), "
                                   f"{workers} host workers + 1 accelerator-model thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def algorithmic_bytes(dec, q_bytes_per_head=D * 4, eq3=False):
    """SURVEY §8d bytes of one step: (metadata, attend) from the device plan.
    eq3: the Eq. 3 upper bound instead -- per-head selected rows summed over
    the group's heads (Σ_h) rather than their union (∪_h), selector.cpp:12."""
    lay = dec.lay
    blk = dec.plan_blk.cpu().numpy()
    kb = dec.plan_kblocks.cpu().numpy()
    bits = dec.sel_bits.cpu().numpy().view(np.uint32)
    s = 2  # bf16
    meta_bytes = 0
    kv_rows = 0
    for b in range(lay.batch):
        for g in range(lay.kv_heads):
            bk = int(blk[b, g])
            defaults = lay.l_sink + lay.l_local + dec.l_new
            kv_rows += defaults
            if bk == 0:
                continue
            nblk = (lay.l_cpu + bk - 1) // bk
            kk = kb[b, g * G:(g + 1) * G]
            if ((kk > 0) & (kk < nblk)).any():
                meta_bytes += nblk * 2 * D * s
            masks = [bits[b, g * G + h] for h in range(G)]
            if not eq3:
                u = np.zeros(bits.shape[-1], np.uint32)
                for m in masks:
                    u |= m
                masks = [u]
            for m in masks:
                sel = np.unpackbits(m.view(np.uint8), bitorder="little")[:nblk].astype(bool)
                ids = np.nonzero(sel)[0]
                lens = np.minimum(bk, lay.l_cpu - ids * bk)
                kv_rows += int(lens.sum())
    heads = lay.batch * H
    attend = kv_rows * 2 * D * s + heads * q_bytes_per_head + heads * (D + 1) * 4
    return meta_bytes, attend


def run_c5(a):
    """configs[4]: 1M-token context, batch 4, the cpu segment split over the
    ranks (context_parallel.py; NCCL all-gathers of the k-th keys, the
    candidates and the (o, lse) partials).  Strong scaling: the job is fixed."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(os.environ.get("FX_BENCH_BACKEND", "nccl"), init_method="env://")
    dev = torch.device("cuda", local)
    from paper_2605_07719_b200.context_parallel import CPShard, TorchComm, cp_decode_step, shard_kv
    from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder

    B, ctx = 4, 1 << 20
    l_cpu = ctx - L_SINK - L_LOCAL
    total = a.warmup + a.steps + 2
    eng = Engine(local)
    full = SparseDecoder(eng, B, HKV, G, D, L_SINK, l_cpu, L_LOCAL, max_new=total, dtype="bf16")
    out = full.generate(dict(seed=1, layers=1, heads=H, group_size=G, head_dim=D, context_len=ctx,
                             decode_steps=total), seeds=[1 + b for b in range(B)], layers=[0] * B,
                        steps=total)
    qs, nk, nv = out["step_q"], out["new_k"], out["new_v"]
    bgt0, ks, st = head_props(B, seed=1)
    props = tuple(torch.as_tensor(x, device=dev) for x in (bgt0, ks, st))
    if world == 1:
        full.build_metadata()
        dec, shards, comm = full, None, None
    else:
        from paper_2605_07719_b200.context_parallel import (PeerShard, PeerTables, cp_decode_step_dist,
                                                            cp_decode_step_peer)
        peer = a.cp_exchange in ("peer", "dist")
        kr = shard_kv(full.k, L_SINK, l_cpu, L_LOCAL, rank, world, total)
        vr = shard_kv(full.v, L_SINK, l_cpu, L_LOCAL, rank, world, total)
        del full
        torch.cuda.empty_cache()
        cls = PeerShard if peer else CPShard
        sh = cls(eng, rank, world, B, HKV, G, D, L_SINK, l_cpu, L_LOCAL, total, "bf16", k=kr, v=vr)
        sh.dec.build_metadata()
        dec, shards = sh.dec, [sh]
        comm = PeerTables.over_dist(eng, sh) if peer else TorchComm()
    step_i = [0]

    def one_step():
        i = step_i[0]
        if shards is None:
            dec.step(qs[i], props=props)
            dec.append(nk[i], nv[i])
        else:
            if a.cp_exchange == "dist":
                cp_decode_step_dist(shards, comm, qs[i], i + 1, props=props)
            elif a.cp_exchange == "peer":
                cp_decode_step_peer(shards, comm, qs[i], i + 1, props=props)
            else:
                cp_decode_step(shards, comm, qs[i], props=props)
            if shards[0].is_last:
                dec.append(nk[i], nv[i])
        step_i[0] += 1

    for _ in range(a.warmup):
        one_step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = eng.launches()
    t0.record()
    for _ in range(a.steps):
        one_step()
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": a.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: the reference's generate(spec) on device, seed 1 + sequence",
            "gpu_launches": int(eng.launches() - n0), "clocks": clk,
            "config": {"workload": "C5: Llama-3-8B layer, 1M ctx, batch 4, per-head budgets from "
                                   "plan_group over the whole sequence",
                       "context": ctx, "global_batch": B, "seq_len": ctx,
                       "parallelism": "single device" if world == 1 else
                       (f"context-parallel x{world}, the selection bracket distributed over peer "
                        f"memory (score ranges, summed histograms, exact-scored bands; CUDA IPC "
                        f"tables, flag waits in the kernels)"
                        if a.cp_exchange == "dist" else
                        f"context-parallel x{world}, one-shot exchanges over peer memory (CUDA IPC "
                        f"tables, flag waits in the select / combine kernels)"
                        if a.cp_exchange == "peer" else
                        f"context-parallel x{world} (all-gathers of k-th keys, candidates, "
                        f"(o, lse))")}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(a):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one rank per GPU; the modulo only matters for a multi-rank smoke test of this
    # code path on a single-GPU box (FX_BENCH_BACKEND=gloo), never for a measurement
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group(os.environ.get("FX_BENCH_BACKEND", "nccl"), init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2605_07719_b200 import _native as N
    from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder

    B = a.batch
    l_cpu = a.context - L_SINK - L_LOCAL
    total_steps = 2 * a.warmup + 5 * a.steps + 8  # timed, graph replay, timing pass, e2e, predictor
    eng = Engine(local)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    shape = (B, HKV, SparseDecoder.cap_rows(a.context, total_steps), D)
    k = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    v = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    if a.data == "normal":  # plain N(0,1) KV, generated on device
        for b in range(B):
            k[b].normal_(generator=gen)
            v[b].normal_(generator=gen)
    dec = SparseDecoder(eng, B, HKV, G, D, L_SINK, l_cpu, L_LOCAL, max_new=total_steps,
                        dtype="bf16", k=k, v=v)
    gen_ms = None
    if a.data == "reference":
        # the reference's generate(spec) (WorkloadSpec defaults: 0.5 streaming / 0.5
        # retrieval heads, one 16-token needle per retrieval head, local boost,
        # drifting decode queries) on the device; entry b = (layer, sequence), the
        # sequence's seed = 1 + its global index
        spec = dict(seed=1, layers=a.layers, heads=H, group_size=G, head_dim=D,
                    context_len=a.context, decode_steps=total_steps)
        seqs = [b % a.seqs for b in range(B)]
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t_gen = time.time()
        out = dec.generate(spec, seeds=[1 + rank * a.seqs + sq for sq in seqs],
                           layers=[b // a.seqs for b in range(B)], steps=total_steps)
        gen_ms = (time.time() - t_gen) * 1e3
        qs = out["step_q"]
        kv_new = torch.stack([out["new_k"], out["new_v"]], dim=1)
        del out
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dec.build_metadata()
    e1.record()
    torch.cuda.synchronize()
    meta_build_ms = e0.elapsed_time(e1)

    bgt0, ks, st = head_props(B, seed=1 + rank)
    props = (torch.as_tensor(bgt0, device=dev), torch.as_tensor(ks, device=dev),
             torch.as_tensor(st, device=dev))
    if a.data == "normal":
        # drifting decode queries (workload.cpp:280-296 recipe), pre-generated on device
        rho = 0.98
        qs = torch.empty((total_steps, B, H, D), dtype=torch.float32, device=dev)
        qs[0].normal_(generator=gen)
        for t in range(1, total_steps):
            noise = torch.randn((B, H, D), generator=gen, device=dev)
            noise = noise / noise.norm(dim=-1, keepdim=True)
            qs[t] = rho * qs[t - 1] / qs[t - 1].norm(dim=-1, keepdim=True) + (1 - rho * rho) ** 0.5 * noise
        qs = qs / qs.norm(dim=-1, keepdim=True) * (D ** 0.5)
        kv_new = torch.randn((total_steps, 2, B, HKV, D), generator=gen, device=dev)

    step_i = [0]

    def one_step():
        # one decode step, then the append of its token (append_new after a step,
        # pipeline.cpp:410-412).  (step(append=...) fuses the append into the next
        # step's plan kernel instead; measured ~1 % slower here, so not used.)
        i = step_i[0]
        dec.step(qs[i], props=props)
        dec.append(kv_new[i, 0], kv_new[i, 1])
        step_i[0] += 1

    for _ in range(a.warmup):
        one_step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = eng.launches()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(a.steps):
        one_step()
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = eng.launches() - n0
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / a.steps
    value = world * a.steps / (ms / 1e3)

    # the same K steps captured once as a CUDA graph (untimed) and replayed:
    # every kernel still runs; only the host launch path leaves the loop
    graph = None
    if not a.quick:
        try:
            s_cap = torch.cuda.Stream(dev)
            g = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s_cap):
                eng.sync_stream()  # the library launches on the capturing stream
                for _ in range(a.steps):
                    one_step()
            eng.sync_stream()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0.record()
            g.replay()
            t1.record()
            torch.cuda.synchronize()
            gms = t0.elapsed_time(t1)
            if world > 1:
                tt = torch.tensor([gms], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                gms = float(tt.item())
            graph = {"value": world * a.steps / (gms / 1e3), "ms_per_step": gms / a.steps,
                     "how": f"{a.steps} steps captured once as one CUDA graph (PDL edges kept), "
                            f"replayed once inside the timed region"}
            del g
        except Exception as e:  # noqa: BLE001
            eng.sync_stream()
            graph = {"value": None, "error": str(e)[:200]}

    result = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
              "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
              "data": ("synthetic: the reference's generate(spec) on device (WorkloadSpec defaults, "
                       "seed 1 + sequence; N(0,1) K/V with planted needles, local boost, drifting "
                       "queries); head properties drawn (seed 1)") if a.data == "reference" else
                      "synthetic (N(0,1) K/V generated on device; head properties drawn, seed 1)",
              "gpu_launches": int(launches), "clocks": clk, "graph_replay": graph}

    if a.quick:
        # profiling runs (ncu): the algorithmic bytes of the attention launch of a
        # few more steps, so a captured launch's DRAM bytes can be set against
        # the bytes it had to move (untimed)
        qb = []
        for _ in range(3):
            one_step()
            torch.cuda.synchronize()
            qb.append(algorithmic_bytes(dec)[1])
        result["quick_attend_bytes_next_steps"] = qb
    if not a.quick:
        # ---- per-kernel CUDA-event timing pass (same steps, same stream) ----
        import ctypes as C
        check = N.check
        check(N.LIB.fx_ctx_reset_timing(eng.ctx))
        check(N.LIB.fx_ctx_set_timing(eng.ctx, 1))
        meta_b = attend_b = 0
        for _ in range(a.steps):
            one_step()
            mb, ab = algorithmic_bytes(dec)
            meta_b += mb
            attend_b += ab
        check(N.LIB.fx_ctx_set_timing(eng.ctx, 0))
        kt = {}
        for i, name in enumerate(N.KERNELS):
            tot, cnt = C.c_double(0), C.c_int64(0)
            check(N.LIB.fx_ctx_kernel_time(eng.ctx, i, C.byref(tot), C.byref(cnt)))
            if cnt.value:
                kt[name] = tot.value / cnt.value
        peak, peak_kind = peaks()
        attend_ms = kt.get("attend", float("nan"))
        achieved = attend_b / a.steps / (attend_ms * 1e-3) / 1e9
        result["roofline"] = {"bound": "hbm", "kernel": "k_attend_tma (K3+K4)",
                              "achieved": achieved, "peak": peak, "unit": "GB/s",
                              "frac": achieved / peak, "peak_kind": peak_kind, "timing": "per-kernel CUDA events in a separate pass with PDL off (events bracket each kernel alone)",
                              "traffic": (ncu_traffic("k_attend", a.workload) or {}).get("dram_bytes_per_launch"),
                              "traffic_launch_algorithmic_bytes": (ncu_traffic("k_attend", a.workload) or {}).get(
                                  "algorithmic_bytes_of_captured_launch"),
                              "algorithmic_bytes_per_launch": attend_b / a.steps}
        score_ms = kt.get("score", float("nan"))
        step_bytes = (meta_b + attend_b) / a.steps
        result["kernels_ms"] = kt
        result["score_kernel"] = {"ms": score_ms, "metadata_bytes": meta_b / a.steps,
                                  "GB/s": meta_b / a.steps / (score_ms * 1e-3) / 1e9}
        result["step_bytes"] = step_bytes
        result["step_GBps"] = step_bytes / (ms_per_step * 1e-3) / 1e9
        # Eq. 3 upper bound of the last step (Σ_h instead of ∪_h): what the
        # per-head reference path would move; the batched K3 reads a block
        # once for all heads of its group
        mb3, ab3 = algorithmic_bytes(dec, eq3=True)
        mb1, ab1 = algorithmic_bytes(dec)
        result["eq3_bytes_last_step"] = {"sum_over_heads": mb3 + ab3, "union_over_heads": mb1 + ab1}

        # ---- end to end: pinned host q / new KV in, o out, every step ----
        if not a.no_e2e:
            qh = qs[: a.steps].cpu().pin_memory()
            kvh = kv_new[: a.steps].cpu().pin_memory()
            oh = torch.empty((a.steps, B, H, D), dtype=torch.float32).pin_memory()
            lh = torch.empty((a.steps, B, H), dtype=torch.float32).pin_memory()
            # a side stream moves step i+1's inputs in and step i's output out
            # while step i computes; every copy is inside the timed region and
            # every step waits for its inputs.  Each step is followed by the
            # append of its token (append_new after a step, pipeline.cpp:410-412);
            # the new-KV rows are triple-buffered.
            qd = [torch.empty((B, H, D), dtype=torch.float32, device=dev) for _ in range(2)]
            kvd = [torch.empty((2, B, HKV, D), dtype=torch.float32, device=dev) for _ in range(3)]
            od = [torch.empty((B, H, D), dtype=torch.float32, device=dev) for _ in range(2)]
            ld = [torch.empty((B, H), dtype=torch.float32, device=dev) for _ in range(2)]
            comp = torch.cuda.current_stream(dev)
            cs = torch.cuda.Stream(dev)
            ev_in = [torch.cuda.Event() for _ in range(2)]
            ev_q = [torch.cuda.Event() for _ in range(2)]   # q buffer consumed
            ev_kv = [torch.cuda.Event() for _ in range(3)]  # new-KV buffer consumed
            ev_out = [torch.cuda.Event() for _ in range(2)]
            ev_read = [torch.cuda.Event() for _ in range(2)]

            def h2d(i):
                with torch.cuda.stream(cs):
                    if i >= 2:
                        cs.wait_event(ev_q[i % 2])    # step i-2 read q buffer i%2
                    if i >= 3:
                        cs.wait_event(ev_kv[i % 3])   # step i-3 appended from kv buffer i%3
                    qd[i % 2].copy_(qh[i], non_blocking=True)
                    kvd[i % 3].copy_(kvh[i], non_blocking=True)
                    ev_in[i % 2].record(cs)

            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0.record()
            h2d(0)
            for i in range(a.steps):
                j = i % 2
                comp.wait_event(ev_in[j])
                if i >= 2:
                    comp.wait_event(ev_read[j])  # output buffer j copied out
                dec.step(qd[j], props=props, out=od[j], lse=ld[j])
                ev_out[j].record(comp)
                dec.append(kvd[i % 3][0], kvd[i % 3][1])  # append_new after the step
                ev_q[j].record(comp)
                ev_kv[i % 3].record(comp)
                if i + 1 < a.steps:
                    h2d(i + 1)
                with torch.cuda.stream(cs):
                    cs.wait_event(ev_out[j])
                    oh[i].copy_(od[j], non_blocking=True)
                    lh[i].copy_(ld[j], non_blocking=True)
                    ev_read[j].record(cs)
            comp.wait_stream(cs)
            t1.record()
            torch.cuda.synchronize()
            ems = t0.elapsed_time(t1)
            if world > 1:
                tt = torch.tensor([ems], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ems = float(tt.item())
            result["e2e"] = {"value": world * a.steps / (ems / 1e3), "unit": UNIT,
                             "h2d_bytes_per_step": int(qd[0].numel() * 4 + kvd[0].numel() * 4),
                             "d2h_bytes_per_step": int(B * H * D * 4 + B * H * 4),
                             "path": "C-ABI fx_decode_step + fx_append_kv per step, pinned "
                                     "host buffers, copies overlapped on a side stream"}

        # ---- predictor-driven plan (C2 as configured: budgets from the predictor) ----
        # prefill_stats once (anchor = the first query), then every step:
        # decode_features -> predict -> plan_group -> select -> attend, all on
        # the device.  Random-init 41->256->384->3 weights (the reference ships
        # no trained model); the output-layer bias is set to the drawn-props
        # operating point (bgt0 ~ 0.03, k ~ 0.005, streaming ~ half).
    if not a.quick and a.workload == "c2":
        from paper_2605_07719_b200.fluxattn import Predictor
        rs = np.random.default_rng(5)
        params = {"w1": rs.standard_normal((256, 41)) * (2.0 / 41) ** 0.5, "b1": np.zeros(256),
                  "w2": rs.standard_normal((384, 256)) * (2.0 / 256) ** 0.5, "b2": np.zeros(384),
                  "w3": rs.standard_normal((3, 384)) * np.array([[1e-4], [2e-5], [1e-2]]),
                  "b3": np.array([0.03, 0.005, 0.0]), "mu": np.zeros(41), "sigma": np.ones(41)}
        e0.record()
        rec = dec.prefill_stats(qs[0], tau=0.10, layer=0)
        e1.record()
        torch.cuda.synchronize()
        prefill_ms = e0.elapsed_time(e1)
        feats = torch.empty((B, H, 41), dtype=torch.float64, device=dev)
        # feature normalization (FeatureNorms, features.cpp:226-233) fitted on the
        # first step's features, as train() does on its training rows
        f0 = dec.decode_features(qs[0], rec, out=feats).reshape(-1, 41)
        params["mu"] = f0.mean(0).cpu().numpy()
        sd = f0.std(0)
        # features constant across heads (layer, lengths, ...) get sigma 0: normalize()
        # passes them through as 0 (features.cpp:226-233)
        params["sigma"] = torch.where(sd > 1e-9 * (1 + f0.mean(0).abs()), sd,
                                      torch.zeros_like(sd)).cpu().numpy()
        pred = Predictor(eng, params)
        z0 = torch.empty((B * H, 3), dtype=torch.float64, device=dev)
        pred(f0, z=z0)  # centre the streaming logit: about half the heads stream
        params["b3"][2] = -float(z0[:, 2].median().item())
        pred.close()
        pred = Predictor(eng, params)

        def pred_step():
            i = step_i[0]
            dec.decode_features(qs[i], rec, out=feats)
            pp = pred(feats)
            dec.step(qs[i], props=pp, append=(kv_new[i - 1, 0], kv_new[i - 1, 1]))
            step_i[0] += 1

        for _ in range(a.warmup):
            pred_step()
        torch.cuda.synchronize()
        t0.record()
        for _ in range(a.steps):
            pred_step()
        t1.record()
        torch.cuda.synchronize()
        pms = t0.elapsed_time(t1)
        # phase split of one more step (events serialize the phases)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        i = step_i[0]
        ev[0].record()
        dec.decode_features(qs[i], rec, out=feats)
        ev[1].record()
        pp = pred(feats)
        ev[2].record()
        dec.step(qs[i], props=pp, append=(kv_new[i - 1, 0], kv_new[i - 1, 1]))
        ev[3].record()
        step_i[0] += 1
        torch.cuda.synchronize()
        stream_frac = float(pp[2].float().mean().item())
        retr_groups = int((dec.plan_blk > 0).sum().item())
        result["predictor_path"] = {
            "value": world * a.steps / (pms / 1e3), "unit": UNIT, "ms_per_step": pms / a.steps,
            "features_ms": ev[0].elapsed_time(ev[1]), "predict_ms": ev[1].elapsed_time(ev[2]),
            "decode_step_ms": ev[2].elapsed_time(ev[3]), "retrieval_groups": retr_groups,
            "prefill_stats_ms": prefill_ms, "streaming_frac": stream_frac,
            "per_step": "fx_decode_features + fx_predict + fx_decode_step + fx_append_kv",
            "model": "random-init 41-256-384-3, output bias at the drawn-props operating point"}
        pred.close()

    result["config"] = {
        "workload": ("C2: Llama-3-8B layer (32q/8kv heads, d128), 128K ctx, batch 16/GPU, "
                     "per-head budgets + per-group granularity (16/32/64/128) from plan_group")
        if a.workload == "c2" else
        ("C4: Llama-3-8B 32-layer decode step, 128K ctx, batch 8/GPU (64 over 8 GPUs), the 32 "
         "layers' (b, g) tasks in one batched step; per-head budgets from plan_group"),
        "layers": a.layers,
        "context": a.context, "global_batch": a.seqs * world, "seq_len": a.context,
        "parallelism": f"batch-sharded x{world} (no collective)", "kv_dtype": "bf16",
        "l2": "per-step working set > 1 GB (inputs larger than the 126 MB L2); no flush",
        "meta_build_ms": meta_build_ms, "generate_ms": gen_ms,
        "budget_source": "drawn head properties (bgt0~U(.01,.05), k~U(0,.01), streaming~B(.5))"}

    # ---- CPU baseline: the compiled reference on a bounded sample (rank 0, N=1) ----
    if rank == 0 and world == 1 and not a.quick and not a.no_cpu_baseline:
        try:
            from oracle.oracle import RefOracle
            ref = RefOracle()
            cores = os.cpu_count() or 1
            workers = max(1, cores - 1)
            kk = dec.k[0, :, : a.context].float().cpu().numpy()
            vv = dec.v[0, :, : a.context].float().cpu().numpy()
            blk = dec.plan_blk[0].cpu().numpy()
            bud = dec.plan_budgets[0].cpu().numpy()
            plans = [None if int(blk[g]) == 0 else (int(blk[g]), bud[g * G:(g + 1) * G])
                     for g in range(HKV)]
            qn = qs[step_i[0] - 1, 0].cpu().numpy()
            times, n_tasks = reference_sample(ref, [(kk[g], vv[g]) for g in range(HKV)], plans,
                                              qn, workers, 5)
            t = min(times) * B
            result["cpu_baseline"] = {
                "value": 1.0 / t, "unit": UNIT, "cores": workers + 1, "kind": "reference",
                "sample": f"1 of {B} sequences ({n_tasks} retrieval-group tasks, same plan and "
                          f"data as the GPU step), best of 5, x{B} extrapolated"}
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                      "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = args_parse()
    if a.impl == "reference":
        run_reference_arm(a)
        return
    if a.workload == "c5":
        run_c5(a)
        return
    run_ours(a)


if __name__ == "__main__":
    main()
