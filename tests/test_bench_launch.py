"""bench.py's launcher and line contract, on CPU (no GPU needed).

`bench.py --gpus N` re-launches itself under torch.distributed.run with one
rank per GPU; --dry-run-launch swaps the decode step for an empty one so the
rank plumbing (WORLD_SIZE check, barriers, max-over-ranks over gloo, the
aggregate value) runs here.  It is a launcher test, never a measurement.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _last_json(out):
    for line in reversed(out.splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    raise AssertionError(f"no JSON line in:\n{out}")


def test_bench_gpus_2_launches_two_ranks():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dry-run-launch", "--steps", "20", "--warmup", "3"],
                       capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line["dry_run"] is True
    assert line["n_gpus"] == 2 and line["ranks"] == 2
    # aggregate over both ranks: 2 x steps / max-over-ranks time of ~1 ms steps
    assert line["value"] > 1.5 * (1e3 / line["ms_per_step"]) * 0.9


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dry-run-launch", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)


def test_both_arms_share_one_config():
    import bench
    for wl in ("c1", "c2", "c3", "c4"):
        a = bench.args_parse(["--workload", wl])
        r = bench.args_parse(["--workload", wl, "--impl", "reference"])
        assert bench.workload_config(a, 1) == bench.workload_config(r, 1)
    a = bench.args_parse([])
    c = bench.workload_config(a, 1)
    assert c["context"] == 131072 and c["global_batch"] == 16 and c["heads"] == 32
    assert bench.args_parse(["--plan", "fixed16"]).plan == "fixed16"
