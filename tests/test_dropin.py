"""The C++ drop-in (include/fluxattn/*.hpp over the C-ABI) used exactly like
the reference API by tests/cpp/dropin_test.cpp; its results are compared with
the CPU oracle on the same inputs (regenerated here from the same LCG)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_DIR = os.path.join(ROOT, "paper_2605_07719_b200", "_lib")


def build_dropin(tmp):
    exe = os.path.join(tmp, "dropin_test")
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L", LIB_DIR,
                    "-lfluxattn_b200", f"-Wl,-rpath,{LIB_DIR}", "-pthread", "-o", exe], check=True)
    return exe


def test_dropin_compiles_against_reference_headers(tmp_path):
    """CPU-only: a reference-API caller compiles and links against the library."""
    build_dropin(str(tmp_path))


class Lcg:
    def __init__(self, s):
        self.s = s

    def next(self):
        self.s = (self.s * 6364136223846793005 + 1442695040888963407) % (1 << 64)
        return np.float32(float((self.s >> 11) & ((1 << 40) - 1)) / float(1 << 40) * 2.0 - 1.0)

    def matrix(self, r, c):
        return np.array([self.next() for _ in range(r * c)], np.float32).reshape(r, c)


@pytest.mark.gpu
def test_dropin_against_oracle(tmp_path, coracle):
    exe = build_dropin(str(tmp_path))
    out = os.path.join(str(tmp_path), "out.json")
    r = subprocess.run([exe, out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    res = json.load(open(out))["cases"]
    D, G, ls, lc, ll = 64, 4, 64, 1500, 256
    g = Lcg(42)
    caches = []
    for _ in range(4):
        parts = [g.matrix(n, D) for n in (ls, ls, lc, lc, ll, ll)]
        nk, nv = g.matrix(2, D), g.matrix(2, D)
        k = np.vstack([parts[0], parts[2], parts[4], nk])
        v = np.vstack([parts[1], parts[3], parts[5], nv])
        caches.append((k, v))
    blks = [16, 32, 64, 128]
    queries = [np.stack([g.matrix(1, D)[0] for _ in range(G)]) for _ in range(4)]
    seg = (ls, lc, ll, 2)
    # per-head case (task 0, head 0)
    ph = res[0]
    k, v = caches[0]
    mins, maxs = coracle.build_metadata(k[ls:ls + lc], 16)
    kb = coracle.blocks_for_budget(0.05, lc, 16)
    want, _ = coracle.topk_blocks(queries[0][0], mins, maxs, kb)
    assert ph["k"] == kb
    assert [int(x) for x in ph["blocks"]] == [int(x) for x in want]
    wo, _, _ = coracle.execute_group(k, v, seg, queries[0][:1], 16, np.array([0.05]))
    assert np.abs(np.array(ph["o"]) - wo[0]).max() < 1e-3
    # run(Executed) over the queue: priority order, outputs per head
    tasks = [c for c in res if c["kind"] == "task"]
    assert [t["group"] for t in tasks] == [10, 11, 12, 13]  # V(blk) descending
    for t in tasks:
        i = t["group"] - 10
        k, v = caches[i]
        wo, _, _ = coracle.execute_group(k, v, seg, queries[i], blks[i],
                                         np.array([0.05, 0.0, 0.2, 1.0]))
        got = np.array([h["o"] for h in t["heads"]])
        assert np.abs(got - wo).max() < 1e-3, (t["group"], np.abs(got - wo).max())


REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _pipeline(name, out, *args):
    exe = os.path.join(REF_DIR, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (make -C oracle dropin, needs /root/reference)")
    r = subprocess.run([exe, out] + [str(a) for a in args], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr + r.stdout
    return json.load(open(out))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [dict(blk=16, bgt=0.1), dict(blk=64, bgt=0.05), dict(blk=0, bgt=0.0)])
def test_reference_pipeline_through_dropin(tmp_path, cfg):
    """The reference's own caller, run_decode (pipeline.cpp:177-415), compiled
    unchanged against include/ and linked to libfluxattn_b200.so, against the
    same program built from the unmodified reference: plans, scheduled tasks
    and the per-head output deviations (sparse vs full attention, both sides
    computed by the implementation under test) agree.  blk 0 = output-aware
    budgets from the reference's label tooling, whose attention now runs on
    the device through the drop-in."""
    args = (4096, 8, 4, 64, 2, 3, cfg["blk"], cfg["bgt"], 1, 7)
    ref = _pipeline("pipeline_ref", str(tmp_path / "ref.json"), *args)
    got = _pipeline("pipeline_dropin", str(tmp_path / "dropin.json"), *args)
    assert len(ref["steps"]) == len(got["steps"]) == 3
    same_plans = sum(a == b for a, b in zip(ref["plans"], got["plans"]))
    if cfg["blk"]:
        assert ref["plans"] == got["plans"]
    else:  # labels from f32 device attention vs f64 host: a boundary flip at most
        assert same_plans >= len(ref["plans"]) - 1, (same_plans, len(ref["plans"]))
    for a, b in zip(ref["steps"], got["steps"]):
        assert a["scheduled_tasks"] == b["scheduled_tasks"]
        assert a["streaming_groups"] == b["streaming_groups"]
        da, db = np.array(a["head_deviations"]), np.array(b["head_deviations"])
        if cfg["blk"] or same_plans == len(ref["plans"]):
            assert np.abs(da - db).max() < 1e-4, np.abs(da - db).max()


@pytest.mark.gpu
def test_reference_pipeline_c2_shape_through_dropin(tmp_path, engine):
    """run_decode at the C2 layer shape (32 q / 8 kv heads, d128, 128K context,
    fixed (16, 0.05)) through the drop-in: the caches stay resident on the
    device between steps (only the appended rows go up, in one batched append),
    so a run(queue, Executed) step costs one fx_decode_step over the f32 caches
    plus the host marshalling -- within 2x of fx_decode_step timed alone (with
    its output read back) on the same shape."""
    import time

    import torch

    from paper_2605_07719_b200.fluxattn import SparseDecoder
    got = _pipeline("pipeline_dropin", str(tmp_path / "c2.json"), 131072, 32, 4, 128, 1, 6, 16, 0.05, 0, 1)
    ms = [s["makespan"] * 1e3 for s in got["steps"]]
    assert all(s["scheduled_tasks"] == 8 for s in got["steps"])
    dec = SparseDecoder(engine, 8, 1, 4, 128, 64, 131072 - 320, 256, max_new=8, dtype="f32")
    dec.k.normal_()
    dec.v.normal_()
    dec.build_metadata()
    q = torch.randn((8, 4, 128), device=engine.device)
    for _ in range(10):
        dec.step(q, fixed=(16, 0.05))
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        o, _ = dec.step(q, fixed=(16, 0.05))
        o.cpu()
    step_ms = (time.perf_counter() - t) / 20 * 1e3
    print("run(queue, Executed) per step (ms):", ["%.3f" % m for m in ms], "fx_decode_step %.3f ms" % step_ms)
    assert max(ms[2:]) < 2.0 * step_ms
    del dec
