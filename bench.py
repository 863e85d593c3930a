#!/usr/bin/env python
"""Fluxion sparse-attention decode step on B200 -- the BASELINE.json metric.

Default workload (BASELINE.json configs[1], "C2"): one Llama-3-8B-shaped decode
layer (32 query / 8 KV heads, head_dim 128), 131072-token context per sequence
(sink 64 | cpu 130752 | local 256 | decoded rows), batch 16 per GPU, bf16 KV
from the reference's generate(spec) run on the device.  Budgets: per-head
properties (bgt0 ~ U(0.01, 0.05), k ~ U(0, 0.01), streaming ~ Bernoulli(0.5),
seed 1; SURVEY §8d perf run) -> on-device plan_group picks each group's
granularity (16/32/64/128) and per-head budgets every step.

One timed step = K5 plan -> K2 score/select (+ fused worklist) -> K3/K4 sparse
GQA attention + fused LSE merge for every head of the batch, plus the append
of the step's new K/V row of every group.  Per-step working set is > 1 GB, far
above the 126 MB L2, so no flush is needed between steps.

Other configs (--workload): c1 (configs[0]: 32K, batch 1, f32, fixed (64,
0.05)), c3 (configs[2]: Qwen 28q/4kv, 256K, batch 8, output-aware budgets
labelled once on the device), c4 (configs[3]: 32 layers x batch 8 per GPU, the
layers' tasks in one batched step), c5 (configs[4]: 1M context, batch 4,
context-parallel over the torchrun ranks).  --plan fixed16: every head
retrieving at (16, 0.05) -- BASELINE.md's 2,015 steps/s target row.

Multi-GPU: `--gpus N` re-launches itself under torch.distributed.run when not
already inside one (one rank per GPU).  C1-C4 shard by batch (weak scaling, no
collective); C5 splits the context (strong scaling).

--impl reference: the reference's own executed CPU path (oracle/_ref, the
unmodified sources compiled here) on the same workload: every sequence of the
batch (for C4 the 8 sequences of one layer, extrapolated x32), data from the
reference's own generate(spec), one run(queue, profile, RunMode::Executed)
per step.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-attn decode steps/s at 128K ctx, bs=16; achieved HBM GB/s vs peak"
UNIT = "steps/s"
D = 128
L_SINK, L_LOCAL = 64, 256

# BASELINE.json configs; `seqs` sequences x `layers` layers per GPU
WORKLOADS = {
    "c1": dict(heads=32, G=4, context=32768, seqs=1, layers=1, dtype="f32", plan="fixed64",
               desc="C1: Llama-3-8B layer (32q/8kv heads, d128), 32K ctx, batch 1, f32 KV"),
    "c2": dict(heads=32, G=4, context=131072, seqs=16, layers=1, dtype="bf16", plan="props",
               desc="C2: Llama-3-8B layer (32q/8kv heads, d128), 128K ctx, batch 16/GPU, bf16 KV"),
    "c3": dict(heads=28, G=7, context=262144, seqs=8, layers=1, dtype="bf16", plan="labels",
               desc="C3: Qwen2.5-7B layer (28q/4kv heads, d128), 256K ctx, batch 8/GPU, bf16 KV"),
    "c4": dict(heads=32, G=4, context=131072, seqs=8, layers=32, dtype="bf16", plan="props",
               desc="C4: Llama-3-8B 32-layer decode step, 128K ctx, batch 8/GPU (64 over 8 GPUs), "
                    "the 32 layers' (b, g) tasks in one batched step, bf16 KV"),
}
PLANS = {
    "props": "drawn head properties (bgt0~U(.01,.05), k~U(0,.01), streaming~B(.5), seed 1) -> "
             "plan_group",
    "fixed16": "fixed (blk 16, budget 0.05) for every head, every head retrieving "
               "(pipeline.cpp:304-311)",
    "fixed64": "fixed (blk 64, budget 0.05) for every head (pipeline.cpp:304-311)",
    "labels": "output-aware oracle head properties (label_streaming / min_budget / fit_curve, "
              "tau 0.10, pipeline.cpp:256-276) of the first decode query -> plan_group",
}


def args_parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--plan", default=None, choices=sorted(PLANS),
                    help="budget source (default: the workload's own)")
    ap.add_argument("--context", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None, help="sequences per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--quick", action="store_true", help="profiling run: timed loop only")
    ap.add_argument("--data", default="reference", choices=["reference", "normal"],
                    help="reference: the reference generator's workload (generate(spec), on "
                         "device); normal: plain N(0,1) K/V")
    ap.add_argument("--cp-exchange", default="dist", choices=["dist", "peer", "collective"],
                    help="c5 exchanges: peer-memory one-shot kernels, or torch.distributed "
                         "all-gathers (NCCL)")
    ap.add_argument("--dry-run-launch", action="store_true",
                    help="launcher self-test without a GPU: ranks, barriers and the max-over-"
                         "ranks reduction over gloo with an empty step (never a measurement)")
    a = ap.parse_args(argv)
    if a.workload != "c5":
        w = WORKLOADS[a.workload]
        a.heads, a.G = w["heads"], w["G"]
        a.hkv = a.heads // a.G
        a.context = a.context or w["context"]
        a.seqs = a.batch or w["seqs"]
        a.layers = w["layers"]
        a.kv_dtype = w["dtype"]
        a.plan = a.plan or w["plan"]
        a.batch = a.layers * a.seqs  # (layer, sequence) entries: independent (b, g) tasks
    return a


def workload_config(a, world):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    return {"workload": f"{WORKLOADS[a.workload]['desc']}; budgets: {PLANS[a.plan]}",
            "heads": a.heads, "kv_heads": a.hkv, "head_dim": D, "layers": a.layers,
            "context": a.context, "seq_len": a.context, "global_batch": a.seqs * world,
            "kv_dtype": a.kv_dtype, "plan": a.plan,
            "data": "the reference's generate(spec), WorkloadSpec defaults, seed 1 + sequence"
            if a.data == "reference" else "N(0,1) K/V",
            "parallelism": f"batch-sharded x{world} (no collective)",
            "l2": "per-step working set > 1 GB (inputs larger than the 126 MB L2); no flush"
            if a.workload != "c1" else "32K f32 working set ~60 MB fits the 126 MB L2 across "
                                       "steps; no flush (launch-bound config)"}


def head_props(batch, heads, seed=1):
    rng = np.random.default_rng(seed)
    bgt0 = rng.uniform(0.01, 0.05, (batch, heads))
    kslope = rng.uniform(0.0, 0.01, (batch, heads))
    streaming = (rng.random((batch, heads)) < 0.5).astype(np.int32)
    return bgt0, kslope, streaming


def fixed_plan(plan):
    return {"fixed16": (16, 0.05), "fixed64": (64, 0.05)}.get(plan)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel, tag):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the
    committed `ncu --set full` extract of the same bench command (profiles/
    ncu_traffic.json for the default c2 line, profiles/ncu_traffic_<tag>.json
    otherwise; written by profiles/summarize_ncu.py); None if absent."""
    name = "ncu_traffic.json" if tag == "c2" else f"ncu_traffic_{tag}.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            t = json.load(f)
        for kname, rec in t["kernels"].items():
            if kernel in kname:
                rec = dict(rec)
                rec["source"] = f"profiles/{name}"
                return rec
    except Exception:
        pass
    return None


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count()}


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
# the reference CPU path (oracle/_ref): run(queue, profile, RunMode::Executed)
# ---------------------------------------------------------------------------
def reference_plans(ref, a, props, fixed, l_cpu, entries):
    """plan_group (selector.cpp:21-46) / the fixed plan (pipeline.cpp:304-311) of
    every (entry, g): None for a streaming group (no task, pipeline.cpp:334-337)."""
    G = a.G
    plans = {}
    for b in entries:
        for g in range(a.hkv):
            if fixed is not None:
                plans[(b, g)] = (fixed[0], np.full(G, fixed[1]))
                continue
            sl = slice(g * G, (g + 1) * G)
            p = ref.plan_group(props[0][b, sl], props[1][b, sl], props[2][b, sl], l_cpu)
            plans[(b, g)] = None if p["streaming_group"] else (p["block_size"], np.asarray(p["budgets"]))
    return plans


def reference_labels(ref, a, data, entries, l_cpu, cores, tau=0.10):
    """Oracle head properties (pipeline.cpp:256-276) with the reference's own
    cache_attention / max_output_norm / label_streaming / min_budget /
    fit_curve, heads in parallel host threads."""
    from concurrent.futures import ThreadPoolExecutor
    seg = (L_SINK, l_cpu, L_LOCAL, 0)
    props = tuple(np.zeros((a.batch, a.heads)) for _ in range(3))
    for b in entries:
        kvs, q = data[b]
        with ThreadPoolExecutor(max_workers=cores) as ex:
            outs = list(ex.map(lambda h: ref.cache_attention(*kvs[h // a.G], seg, q[h]),
                               range(a.heads)))
        nrm = ref.max_output_norm(np.stack(outs))

        def label(h):
            k, v = kvs[h // a.G]
            if ref.label_streaming(k, v, seg, q[h], outs[h], nrm, tau):
                return 0.0, 0.0, 1
            buds = [ref.min_budget(k, v, seg, q[h], blk, outs[h], nrm, tau)[0]
                    for blk in (1, 16, 32, 64, 128)]
            kk, _, _ = ref.fit_curve([16, 32, 64, 128], buds[1:], buds[0], False)
            return buds[0], kk, 0

        with ThreadPoolExecutor(max_workers=cores) as ex:
            for h, (b0, kk, st) in enumerate(ex.map(label, range(a.heads))):
                props[0][b, h], props[1][b, h], props[2][b, h] = b0, kk, st
    return props[0], props[1], props[2].astype(np.int32)


def reference_run(ref, batch, workers, repeats, want_outputs=False):
    """`repeats` executed runs of the whole queue; per-run wall seconds."""
    times, out = [], None
    for i in range(repeats):
        sec, o = batch.run(workers, want_outputs=want_outputs and i == repeats - 1)
        times.append(sec)
        if o is not None:
            out = o
    return times, out


def run_reference_arm(a):
    """--impl reference: the reference CPU path on rank 0; other ranks exit."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import RefOracle
    ref = RefOracle()
    ci = cpu_info()
    cores = ci["nproc"] or 1
    workers = max(1, cores - 1)
    if a.workload == "c5":
        print(json.dumps({"impl": "reference", "unavailable": "C5 (1M context) reference run "
                          "would need ~70 GB of f32 host KV per step sample; use --workload c2"}))
        return
    l_cpu = a.context - L_SINK - L_LOCAL
    # C4: the 8 sequences of layer 0 (64 tasks; every layer is the same shape) x32
    entries = list(range(a.seqs)) if a.workload == "c4" else list(range(a.batch))
    scale = a.batch / len(entries)
    t_gen = time.time()

    def gen(b):
        seq = b % a.seqs
        layer = b // a.seqs
        if a.data == "reference":
            w = ref.generate(seed=1 + seq, layers=layer + 1, heads=a.heads, group_size=a.G,
                             head_dim=D, context_len=a.context, decode_steps=1)
            return [w.group_kv(layer, g) for g in range(a.hkv)], w.queries(layer, 0)
        rng = np.random.default_rng(1 + b)
        kv = [(rng.standard_normal((a.context, D), dtype=np.float32),
               rng.standard_normal((a.context, D), dtype=np.float32)) for _ in range(a.hkv)]
        q = rng.standard_normal((a.heads, D)).astype(np.float32)
        return kv, q * (np.sqrt(D) / np.linalg.norm(q, axis=-1, keepdims=True))

    with ThreadPoolExecutor(max_workers=min(len(entries), cores)) as ex:
        data = dict(zip(entries, ex.map(gen, entries)))
    gen_s = time.time() - t_gen
    fixed = fixed_plan(a.plan)
    props = head_props(a.batch, a.heads, seed=1)
    if a.plan == "labels":  # the reference's own oracle labels of the first decode query
        props = reference_labels(ref, a, data, entries, l_cpu, cores)
    plans = reference_plans(ref, a, props, fixed, l_cpu, entries)
    batch = ref.batch()
    meta_s = 0.0
    n_tasks = 0
    for b in entries:
        kvs, q = data[b]
        for g in range(a.hkv):
            if plans[(b, g)] is None:
                continue
            blk, bud = plans[(b, g)]
            meta_s += batch.add(kvs[g][0], kvs[g][1], (L_SINK, l_cpu, L_LOCAL, 0),
                                q[g * a.G:(g + 1) * a.G], blk, bud)
            n_tasks += 1
        data[b] = None  # the batch holds its own copy
    times, _ = reference_run(ref, batch, workers, a.warmup + a.steps)
    timed = times[a.warmup:] if len(times) > a.warmup else times
    best = min(timed) * scale
    mean = float(np.mean(timed)) * scale
    value = 1.0 / best
    sample = (f"every sequence of the batch: {n_tasks} retrieval-group tasks of {len(entries)} "
              f"entries per step" + (f", x{scale:g} for the {a.layers} layers" if scale != 1 else "")
              + f"; run(queue, profile, RunMode::Executed) with {workers} host workers + 1 "
                f"accelerator-model thread; value = best of {len(timed)} timed runs "
                f"(BASELINE.md §2), mean {1.0 / mean:.3g} steps/s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": best * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: " + workload_config(a, 1)["data"],
        "config": workload_config(a, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers + 1, "kind": "reference",
                         "sample": sample, "cpu_model": ci["model"], "nproc": ci["nproc"],
                         "mean_value": 1.0 / mean, "generate_s": gen_s,
                         "metadata_build_s": meta_s},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_and_parity(a, dec, q, o, lse, plan_step, ref_runs=5, parity=True, entries=None):
    """The compiled reference on the GPU step's exact data (bf16 bits upcast to
    f32, the same plan and queries, the same decoded rows): whole batch (C4: one
    layer's 8 sequences, x32), best of `ref_runs` executed runs.  Then parity of
    that step: the reference's outputs vs ours for every task, every head's
    selection vs the C restatement's topk_blocks, every plan vs plan_group."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    from oracle.oracle import COracle, RefOracle
    ref = RefOracle()
    ci = cpu_info()
    cores = ci["nproc"] or 1
    workers = max(1, cores - 1)
    lay = dec.lay
    G, hkv = lay.group_size, lay.kv_heads
    l_cpu, l_new = lay.l_cpu, dec.l_new
    n_rows = lay.l_sink + l_cpu + lay.l_local + l_new
    seg = (lay.l_sink, l_cpu, lay.l_local, l_new)
    if entries is None:
        entries = list(range(a.seqs)) if a.workload == "c4" else list(range(lay.batch))
    scale = lay.batch / len(entries)
    blk = dec.plan_blk.cpu().numpy()
    bud = dec.plan_budgets.cpu().numpy()
    kbl = dec.plan_kblocks.cpu().numpy()
    bits = dec.sel_bits.cpu().numpy().view(np.uint32)
    qn = q.cpu().numpy()
    on, ln = o.cpu().numpy(), lse.cpu().numpy()
    batch = ref.batch()
    tasks = []
    for b in entries:
        for g in range(hkv):
            if int(blk[b, g]) == 0:
                continue
            k = dec.k[b, g, :n_rows].float().cpu().numpy()
            v = dec.v[b, g, :n_rows].float().cpu().numpy()
            batch.add(k, v, seg, qn[b, g * G:(g + 1) * G], int(blk[b, g]), bud[b, g * G:(g + 1) * G])
            tasks.append((b, g))
    times, ro = reference_run(ref, batch, workers, ref_runs, want_outputs=parity)
    t = min(times) * scale
    res = {"value": 1.0 / t, "unit": UNIT, "cores": workers + 1, "kind": "reference",
           "cpu_model": ci["model"], "nproc": ci["nproc"],
           "sample": f"{len(tasks)} retrieval-group tasks = every (b, g) of "
                     + (f"{len(entries)} of the {lay.batch} batch entries, x{scale:g}"
                        if scale != 1 else f"all {len(entries)} sequences")
                     + f" (the GPU step's data, plan and queries), run(queue, profile, "
                       f"RunMode::Executed) with {workers} host workers + 1 accelerator-model "
                       f"thread, best of {ref_runs}",
           "mean_value": 1.0 / (float(np.mean(times)) * scale)}
    if not parity:
        return res, None
    # ---- parity of the step against the reference / the C restatement ----
    errs = []
    for i, (b, g) in enumerate(tasks):
        want = ro[i]
        got = on[b, g * G:(g + 1) * G]
        errs.append(float(np.abs(got - want).max() / max(1.0, np.abs(want).max())))
    corc = COracle()

    def sel_check(bg):
        b, g = bg
        bk = int(blk[b, g])
        k_cpu = dec_kcpu[bg]
        mins, maxs = corc.build_metadata(k_cpu, bk)
        nblk = mins.shape[0]
        mism = 0
        for hg in range(G):
            h = g * G + hg
            want, _ = corc.topk_blocks(qn[b, h], mins, maxs, int(kbl[b, h]))
            got = np.nonzero(np.unpackbits(bits[b, h].view(np.uint8), bitorder="little")[:nblk])[0]
            if not np.array_equal(np.sort(want.astype(np.int64)), got):
                mism += 1
        return mism

    dec_kcpu = {}
    for bg in tasks:
        b, g = bg
        dec_kcpu[bg] = dec.k[b, g, lay.l_sink:lay.l_sink + l_cpu].float().cpu().numpy()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        mism = sum(ex.map(sel_check, tasks))
    plan_mism = 0
    if plan_step is not None:
        for b in entries:
            for g in range(hkv):
                sl = slice(g * G, (g + 1) * G)
                p = ref.plan_group(plan_step[0][b, sl], plan_step[1][b, sl], plan_step[2][b, sl], l_cpu)
                want_blk = 0 if p["streaming_group"] else p["block_size"]
                if int(blk[b, g]) != want_blk or (want_blk and not np.array_equal(bud[b, sl], p["budgets"])):
                    plan_mism += 1
    par = {"tasks": len(tasks), "heads": len(tasks) * G, "max_rel_err": max(errs) if errs else 0.0,
           "tolerance": 2e-2 if lay.dtype == 1 else 1e-3,
           "selection_mismatches": int(mism), "plan_mismatches": int(plan_mism),
           "against": "outputs: the compiled reference's run(Executed) results of the same step; "
                      "selections: the C restatement's topk_blocks of every head (oracle/"
                      "fx_oracle.c, pinned to the reference); plans: the reference's plan_group",
           "lse_finite": bool(np.isfinite(ln).all())}
    return res, par


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def algorithmic_bytes(dec, q_bytes_per_head=D * 4, eq3=False):
    """SURVEY §8d bytes of one step: (metadata, attend) from the device plan.
    eq3: the Eq. 3 upper bound instead -- per-head selected rows summed over
    the group's heads (Σ_h) rather than their union (∪_h), selector.cpp:12."""
    lay = dec.lay
    G = lay.group_size
    blk = dec.plan_blk.cpu().numpy()
    kb = dec.plan_kblocks.cpu().numpy()
    bits = dec.sel_bits.cpu().numpy().view(np.uint32)
    s = 2 if lay.dtype == 1 else 4
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
                meta_bytes += nblk * 2 * lay.head_dim * s
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
    heads = lay.batch * dec.heads
    attend = kv_rows * 2 * lay.head_dim * s + heads * q_bytes_per_head + heads * (lay.head_dim + 1) * 4
    return meta_bytes, attend


def run_c5(a):
    """configs[4]: 1M-token context, batch 4, the cpu segment split over the
    ranks (context_parallel.py).  Strong scaling: the job is fixed."""
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

    H, HKV, G = 32, 8, 4
    B, ctx = 4, 1 << 20
    l_cpu = ctx - L_SINK - L_LOCAL
    total = a.warmup + 2 * a.steps + 4
    eng = Engine(local)
    full = SparseDecoder(eng, B, HKV, G, D, L_SINK, l_cpu, L_LOCAL, max_new=total, dtype="bf16")
    out = full.generate(dict(seed=1, layers=1, heads=H, group_size=G, head_dim=D, context_len=ctx,
                             decode_steps=total), seeds=[1 + b for b in range(B)], layers=[0] * B,
                        steps=total)
    qs, nk, nv = out["step_q"], out["new_k"], out["new_v"]
    bgt0, ks, st = head_props(B, H, seed=1)
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
    result = {
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
                    f"(o, lse))")}}
    if world == 1 and not a.quick:
        import ctypes as C

        from paper_2605_07719_b200 import _native as N
        N.check(N.LIB.fx_ctx_reset_timing(eng.ctx))
        N.check(N.LIB.fx_ctx_set_timing(eng.ctx, 1))
        attend_b = meta_b = 0
        for _ in range(a.steps):
            one_step()
            mb, ab = algorithmic_bytes(dec)
            meta_b += mb
            attend_b += ab
        N.check(N.LIB.fx_ctx_set_timing(eng.ctx, 0))
        kt = {}
        for i, name in enumerate(N.KERNELS):
            tot, cnt = C.c_double(0), C.c_int64(0)
            N.check(N.LIB.fx_ctx_kernel_time(eng.ctx, i, C.byref(tot), C.byref(cnt)))
            if cnt.value:
                kt[name] = tot.value / cnt.value
        peak, peak_kind = peaks()
        achieved = attend_b / a.steps / (kt["attend"] * 1e-3) / 1e9
        tr = ncu_traffic("k_attend", "c5")
        result["roofline"] = {"bound": "hbm", "kernel": "k_attend_tma (K3 with its per-unit epilogue; "
                              "the unit-partial merge kernel is kernels_ms.merge)", "achieved": achieved,
                              "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                              "peak_kind": peak_kind, "traffic": (tr or {}).get("dram_bytes_per_launch"),
                              "traffic_source": (tr or {}).get("source"),
                              "algorithmic_bytes_per_launch": attend_b / a.steps}
        result["kernels_ms"] = kt
        step_bytes = (meta_b + attend_b) / a.steps
        result["step_bytes"] = step_bytes
        result["step_GBps"] = step_bytes / (result["ms_per_step"] * 1e-3) / 1e9
        # e2e: pinned host q in, o + lse out, per step, through the C-ABI; a side
        # stream moves step i+1's q in and step i's output out while step i
        # computes (double-buffered), every copy inside the timed region
        qh = qs[: a.steps].cpu().pin_memory()
        oh = torch.empty((a.steps, B, H, D), dtype=torch.float32).pin_memory()
        lh = torch.empty((a.steps, B, H), dtype=torch.float32).pin_memory()
        qd = [torch.empty((B, H, D), dtype=torch.float32, device=dev) for _ in range(2)]
        od = [torch.empty((B, H, D), dtype=torch.float32, device=dev) for _ in range(2)]
        ld = [torch.empty((B, H), dtype=torch.float32, device=dev) for _ in range(2)]
        comp = torch.cuda.current_stream(dev)
        cs = torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_q = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev_read = [torch.cuda.Event() for _ in range(2)]

        def h2d(i):
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(ev_q[i % 2])  # step i-2 read q buffer i%2
                qd[i % 2].copy_(qh[i], non_blocking=True)
                ev_in[i % 2].record(cs)

        torch.cuda.synchronize()
        t0.record()
        h2d(0)
        for i in range(a.steps):
            j = i % 2
            comp.wait_event(ev_in[j])
            if i >= 2:
                comp.wait_event(ev_read[j])  # output buffer j copied out
            dec.step(qd[j], props=props, out=od[j], lse=ld[j])
            ev_out[j].record(comp)
            ev_q[j].record(comp)
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
        result["e2e"] = {"value": a.steps / (ems / 1e3), "unit": UNIT,
                         "h2d_bytes_per_step": B * H * D * 4, "d2h_bytes_per_step": B * H * (D + 1) * 4,
                         "path": "C-ABI fx_decode_step per step, pinned host q in, o + lse out, "
                                 "copies overlapped on a side stream (double-buffered)"}
        if not a.no_cpu_baseline:  # the reference on 1 of the 4 sequences (8 GB of f32 KV), x4
            try:
                q_par = qs[step_i[0]].contiguous()
                o_par, lse_par = dec.step(q_par, props=props)
                torch.cuda.synchronize()
                a.workload, a.seqs = "c5", B
                cb, par = cpu_baseline_and_parity(a, dec, q_par, o_par.clone(), lse_par.clone(),
                                                  (bgt0, ks, st), ref_runs=3, entries=[0])
                result["cpu_baseline"] = cb
                if par is not None:
                    result["parity"] = par
            except Exception as e:  # noqa: BLE001
                result["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                          "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(a):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"bench: --gpus {a.gpus} but WORLD_SIZE={world}; run `bench.py --gpus N` "
                         f"(it launches N ranks itself) or torchrun with --nproc-per-node N")
    # one rank per GPU; the modulo only matters for a multi-rank smoke test of this
    # code path on a single-GPU box (FX_BENCH_BACKEND=gloo), never for a measurement
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(os.environ.get("FX_BENCH_BACKEND", "nccl"), init_method="env://")
    dev = torch.device("cuda", local)

    from paper_2605_07719_b200 import _native as N
    from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder

    B, H, HKV, G = a.batch, a.heads, a.hkv, a.G
    l_cpu = a.context - L_SINK - L_LOCAL
    total_steps = 2 * a.warmup + 5 * a.steps + 60 + (200 if os.environ.get("FX_BENCH_PRED_DIAG") else 0)
    eng = Engine(local)
    tdt = torch.bfloat16 if a.kv_dtype == "bf16" else torch.float32
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    shape = (B, HKV, SparseDecoder.cap_rows(a.context, total_steps), D)
    k = torch.empty(shape, dtype=tdt, device=dev)
    v = torch.empty(shape, dtype=tdt, device=dev)
    if a.data == "normal":  # plain N(0,1) KV, generated on device
        for b in range(B):
            k[b].normal_(generator=gen)
            v[b].normal_(generator=gen)
    dec = SparseDecoder(eng, B, HKV, G, D, L_SINK, l_cpu, L_LOCAL, max_new=total_steps,
                        dtype=a.kv_dtype, k=k, v=v)
    gen_ms = None
    anchor = None
    if a.data == "reference":
        # the reference's generate(spec) (WorkloadSpec defaults: 0.5 streaming / 0.5
        # retrieval heads, one 16-token needle per retrieval head, local boost,
        # drifting decode queries) on the device; entry b = (layer, sequence), the
        # sequence's seed = 1 + its global index
        spec = dict(seed=1, layers=a.layers, heads=H, group_size=G, head_dim=D,
                    context_len=a.context, decode_steps=total_steps)
        t_gen = time.time()
        out = dec.generate(spec, seeds=[1 + rank * a.seqs + b % a.seqs for b in range(B)],
                           layers=[b // a.seqs for b in range(B)], steps=total_steps)
        gen_ms = (time.time() - t_gen) * 1e3
        qs = out["step_q"]
        anchor = out["anchor"]
        kv_new = torch.stack([out["new_k"], out["new_v"]], dim=1)
        del out
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dec.build_metadata()  # first call: module load (lazy loading) and attribute setup
    torch.cuda.synchronize()
    e0.record()
    dec.build_metadata()  # timed: the same levels rebuilt from the same K
    e1.record()
    torch.cuda.synchronize()
    meta_build_ms = e0.elapsed_time(e1)

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
        anchor = qs[0]

    fixed = fixed_plan(a.plan)
    label_ms = None
    props_host = None
    if a.plan == "labels":
        # output-aware budgets (pipeline.cpp:256-276) of the first decode query,
        # labelled once on the device and fed to plan_group every step
        e0.record()
        lab = dec.label_heads(qs[0], tau=0.10)
        e1.record()
        torch.cuda.synchronize()
        label_ms = e0.elapsed_time(e1)
        props = (lab["bgt0"], lab["kslope"], lab["streaming"])
        props_host = tuple(t.cpu().numpy() for t in props)
    elif fixed is None:
        props_host = head_props(B, H, seed=1 + rank)
        props = tuple(torch.as_tensor(x, device=dev) for x in props_host)
    else:
        props = None
    plan_kw = dict(fixed=fixed) if fixed is not None else dict(props=props)

    step_i = [0]

    def one_step():
        # one decode step; the previous step's token (append_new after a step,
        # pipeline.cpp:410-412) is appended inside this step's first kernel
        i = step_i[0]
        ap = (kv_new[i - 1, 0], kv_new[i - 1, 1]) if i > 0 else None
        dec.step(qs[i], append=ap, **plan_kw)
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

    def max_over_ranks(x):
        if world > 1:
            tt = torch.tensor([x], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt.item())
        return x

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
            gms = max_over_ranks(t0.elapsed_time(t1))
            graph = {"value": world * a.steps / (gms / 1e3), "ms_per_step": gms / a.steps,
                     "how": f"{a.steps} steps captured once as one CUDA graph (PDL edges kept), "
                            f"replayed once inside the timed region"}
            del g
        except Exception as e:  # noqa: BLE001
            eng.sync_stream()
            graph = {"value": None, "error": str(e)[:200]}

    result = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
              "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
              "dtype": a.kv_dtype,
              "data": ("synthetic: the reference's generate(spec) on device (WorkloadSpec defaults, "
                       "seed 1 + sequence; N(0,1) K/V with planted needles, local boost, drifting "
                       "queries)") if a.data == "reference" else
                      "synthetic (N(0,1) K/V generated on device)",
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
        tag = a.workload if a.plan == WORKLOADS[a.workload]["plan"] else f"{a.workload}_{a.plan}"
        tr = ncu_traffic("k_attend", tag)
        kname = ("k_attend_tma (K3 with its per-unit epilogue; the unit-partial merge kernel is "
                 "kernels_ms.merge)") if a.kv_dtype == "bf16" else ("k_attend_f32w (K3, f32 warp streams; the "
                                                                    "chunk merge is kernels_ms.merge)")
        result["roofline"] = {"bound": "hbm", "kernel": kname,
                              "achieved": achieved, "peak": peak, "unit": "GB/s",
                              "frac": achieved / peak, "peak_kind": peak_kind,
                              "timing": "per-kernel CUDA events on the ctx stream in a separate pass "
                                        "over the same workload, PDL off (events bracket each kernel "
                                        "alone)",
                              "traffic": (tr or {}).get("dram_bytes_per_launch"),
                              "traffic_source": (tr or {}).get("source"),
                              "traffic_launch_algorithmic_bytes": (tr or {}).get(
                                  "algorithmic_bytes_of_captured_launch"),
                              "algorithmic_bytes_per_launch": attend_b / a.steps}
        score_ms = kt.get("score", float("nan"))
        step_bytes = (meta_b + attend_b) / a.steps
        result["kernels_ms"] = kt
        result["score_kernel"] = {"ms": score_ms, "metadata_bytes": meta_b / a.steps,
                                  "GB/s": meta_b / a.steps / (score_ms * 1e-3) / 1e9 if meta_b else None}
        result["step_bytes"] = step_bytes
        result["step_GBps"] = step_bytes / (ms_per_step * 1e-3) / 1e9
        result["step_frac_of_peak"] = result["step_GBps"] / peak
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
                        cs.wait_event(ev_kv[i % 3])   # step i-2 appended kv_{i-3} from buffer i%3
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
                # the previous step's token is appended inside this step (append_new)
                ap = (kvd[(i - 1) % 3][0], kvd[(i - 1) % 3][1]) if i > 0 else None
                dec.step(qd[j], out=od[j], lse=ld[j], append=ap, **plan_kw)
                ev_out[j].record(comp)
                ev_q[j].record(comp)
                if i > 0:
                    ev_kv[(i - 1) % 3].record(comp)
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
            ems = max_over_ranks(t0.elapsed_time(t1))
            result["e2e"] = {"value": world * a.steps / (ems / 1e3), "unit": UNIT,
                             "h2d_bytes_per_step": int(qd[0].numel() * 4 + kvd[0].numel() * 4),
                             "d2h_bytes_per_step": int(B * H * D * 4 + B * H * 4),
                             "path": "C-ABI fx_decode_step per step (the previous token's append "
                                     "fused), pinned host buffers, copies overlapped on a side stream"}

    # ---- predictor-driven plan (C2 as configured: budgets from the predictor) ----
    # prefill_stats once (anchor = the generator's prefill query), then every step:
    # decode_features -> predict -> plan_group -> select -> attend, all on the
    # device.  Random-init 41->256->384->3 weights (the reference ships no
    # trained model); the output-layer bias is set to the drawn-props operating
    # point (bgt0 ~ 0.03, k ~ 0.005, streaming ~ half).
    if not a.quick and a.workload == "c2" and a.plan == "props":
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
            # the previous token is appended inside the feature kernel (the
            # features see it, as decode_features after append_new does)
            i = step_i[0]
            pp = dec.predict_props(qs[i], rec, pred, append=(kv_new[i - 1, 0], kv_new[i - 1, 1]))
            dec.step(qs[i], props=pp)
            step_i[0] += 1
            return pp

        for _ in range(a.warmup):
            pred_step()
        torch.cuda.synchronize()
        t0.record()
        for _ in range(a.steps):
            pp = pred_step()
        t1.record()
        torch.cuda.synchronize()
        pms = max_over_ranks(t0.elapsed_time(t1))
        if os.environ.get("FX_BENCH_PRED_DIAG"):  # loop-structure diagnostics (stderr)
            def loop_ms(fn, n=40):
                torch.cuda.synchronize()
                t0.record()
                for _ in range(n):
                    fn()
                t1.record()
                torch.cuda.synchronize()
                return t0.elapsed_time(t1) / n

            def step_noappend():
                i = step_i[0]
                dec.step(qs[i], props=dec.predict_props(qs[i], rec, pred))
                step_i[0] += 1

            def step_split_append():
                i = step_i[0]
                dec.append(kv_new[i - 1, 0], kv_new[i - 1, 1])
                dec.step(qs[i], props=dec.predict_props(qs[i], rec, pred))
                step_i[0] += 1

            def props_only():
                i = step_i[0]
                dec.predict_props(qs[i], rec, pred)

            def step_only():
                i = step_i[0]
                dec.step(qs[i], props=pp)

            for nm, fn in [("pred_step", pred_step), ("no_append", step_noappend),
                           ("separate_append", step_split_append), ("props_only", props_only),
                           ("step_only", step_only), ("pred_step_again", pred_step)]:
                print(f"pred diag {nm}: {loop_ms(fn):.4f} ms/iter (l_new {dec.l_new})", file=sys.stderr, flush=True)
        # per-step split of 40 more steps (events around each call, synchronized
        # per step): the plan the predictor produces changes with the decoded rows
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        split = []
        for _ in range(40):
            i = step_i[0]
            evs[0].record()
            pp = dec.predict_props(qs[i], rec, pred, append=(kv_new[i - 1, 0], kv_new[i - 1, 1]))
            evs[1].record()
            dec.step(qs[i], props=pp)
            evs[2].record()
            step_i[0] += 1
            torch.cuda.synchronize()
            split.append((evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(evs[2]),
                          int((dec.plan_blk > 0).sum().item())))
        split = np.array(split)
        # phase split: the props launch alone and the step alone, each repeated
        # back to back on the same inputs (no append), CUDA events around the loop
        nrep = 20
        i = step_i[0]
        t0.record()
        for _ in range(nrep):
            pp = dec.predict_props(qs[i], rec, pred)
        t1.record()
        torch.cuda.synchronize()
        props_ms = t0.elapsed_time(t1) / nrep
        t0.record()
        for _ in range(nrep):
            dec.step(qs[i], props=pp)
        t1.record()
        torch.cuda.synchronize()
        pstep_ms = t0.elapsed_time(t1) / nrep
        stream_frac = float(pp[2].float().mean().item())
        retr_groups = int((dec.plan_blk > 0).sum().item())
        # bytes of the step on the predictor's plan (same formula as
        # step_bytes): the predictor's plan is a different, heavier plan than the
        # drawn properties' (more retrieval heads), so compare HBM fractions
        pmb, pab = algorithmic_bytes(dec)
        ppeak, _ = peaks()
        result["predictor_path"] = {
            "value": world * a.steps / (pms / 1e3), "unit": UNIT, "ms_per_step": pms / a.steps,
            "predict_props_ms": props_ms, "decode_step_ms": pstep_ms, "decoded_rows": dec.l_new,
            "per_step_split": {"steps": len(split), "props_ms_median": float(np.median(split[:, 0])),
                               "step_ms_median": float(np.median(split[:, 1])),
                               "step_ms_p90": float(np.percentile(split[:, 1], 90)),
                               "step_ms_max": float(split[:, 1].max()),
                               "retrieval_groups_min": int(split[:, 2].min()),
                               "retrieval_groups_max": int(split[:, 2].max())},
            "retrieval_groups": retr_groups,
            "decode_step_bytes": pmb + pab,
            "decode_step_frac_of_peak": (pmb + pab) / (pstep_ms * 1e-3) / 1e9 / ppeak,
            "prefill_stats_ms": prefill_ms, "streaming_frac": stream_frac,
            "per_step": "fx_predict_props (previous token appended; decode features as chunk "
                        "partials + one clustered merge with layer 1; layers 2 + 3) + fx_decode_step",
            "model": "random-init 41-256-384-3, output bias at the drawn-props operating point"}
        pred.close()

    result["config"] = workload_config(a, world)
    result["setup"] = {"meta_build_ms": meta_build_ms, "generate_ms": gen_ms,
                       "label_ms": label_ms}

    # ---- CPU baseline + in-run parity: the compiled reference on this step's data ----
    if rank == 0 and world == 1 and not a.quick and not a.no_cpu_baseline:
        try:
            # one more step without its append: the step the reference re-runs
            i = step_i[0]
            q_par = qs[i].contiguous()
            o_par, lse_par = dec.step(q_par, **plan_kw)
            torch.cuda.synchronize()
            o_par, lse_par = o_par.clone(), lse_par.clone()
            cb, par = cpu_baseline_and_parity(a, dec, q_par, o_par, lse_par, props_host,
                                              parity=not a.no_parity)
            result["cpu_baseline"] = cb
            if par is not None:
                result["parity"] = par
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                      "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_dry_launch(a):
    """Launcher self-test (CPU, gloo): every rank times an empty step; the
    max-over-ranks reduction and the aggregate follow the real arm.  The line
    says dry_run -- it is never a measurement."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"bench: --gpus {a.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    for _ in range(a.warmup):
        time.sleep(0.001)
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    for _ in range(a.steps):
        time.sleep(0.001)
    ms = (time.perf_counter() - t) * 1e3
    if world > 1:
        tt = torch.tensor([ms])
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "ranks": world,
                          "value": world * a.steps / (ms / 1e3), "unit": UNIT,
                          "ms_per_step": ms / a.steps, "steps": a.steps, "warmup": a.warmup}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    a = args_parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
               "--nproc-per-node", str(a.gpus), "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        env = dict(os.environ)
        if a.impl == "ours" and not a.dry_run_launch:
            env.setdefault("NCCL_DEBUG", "INFO")
            env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        sys.exit(subprocess.call(cmd, env=env))
    # Python's cyclic collector off for the run: a gen-2 pass inside an
    # unsynchronized timed loop stalls the launching thread and drains the GPU
    # (reference counting still frees everything the loops allocate)
    gc.collect()
    gc.disable()
    if a.dry_run_launch:
        run_dry_launch(a)
        return
    if a.impl == "reference":
        run_reference_arm(a)
        return
    if a.workload == "c5":
        run_c5(a)
        return
    run_ours(a)


if __name__ == "__main__":
    main()
