"""bench.py --impl reference (the fp64 oracle timed on host cores) on CPU: the JSON-line
contract of the reference arm, and non-zero ranks exiting without work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env=None, *extra):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--config", "cfg1", "--steps", "2", "--warmup", "1", *extra],
                          capture_output=True, text=True, timeout=300, cwd=ROOT, env=e)


def test_reference_arm_json_line():
    out = _run()
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    out = _run({"RANK": "1", "WORLD_SIZE": "2"})
    assert out.returncode == 0, out.stderr[-2000:]
    assert not [l for l in out.stdout.splitlines() if l.startswith("{")]


def _clean_env(extra=None):
    e = {k: v for k, v in os.environ.items()
         if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    e.update(extra or {})
    return e


def test_gpus_flag_launches_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run:
    two processes with RANK / LOCAL_RANK 0 and 1 and WORLD_SIZE 2; only rank 0 prints the
    JSON line, which reports n_gpus = 2."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                          "reference", "--config", "cfg1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=_clean_env({"SKEI_BENCH_RANKINFO": "1"}))
    assert out.returncode == 0, out.stderr[-2000:]
    info = sorted(l.split()[1:] for l in out.stderr.splitlines() if l.startswith("rankinfo"))
    assert info == [["rank=0", "local=0", "world=2"], ["rank=1", "local=1", "world=2"]], out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_gpus_flag_must_match_world_size():
    out = _run({"RANK": "0", "WORLD_SIZE": "2"}, "--gpus", "4")
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr


def test_reference_arm_steps_fit_its_run_time():
    """Every reference step is one whole pass of the batch: steps x ms_per_step is time the
    process really spent (the driver's fits_in_driver_run check)."""
    import time
    t0 = time.perf_counter()
    out = _run(_clean_env())
    wall = time.perf_counter() - t0
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert d["steps"] * d["ms_per_step"] * 1e-3 <= wall
    assert "whole" in d["cpu_baseline"]["sample"] and d["cpu_baseline"]["host_cores"] >= 1


def test_link_probe_two_ranks_gloo():
    """tools/link_probe.py (SURVEY M2 interconnect probes) under torch.distributed.run with two
    gloo ranks: rank 0 alone prints one JSON line with the all-reduce, all-gather and
    point-to-point entries (the numbers are meaningless on CPU)."""
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                          "29547", os.path.join(ROOT, "tools", "link_probe.py"), "--iters", "1",
                          "--backend", "gloo", "--bytes", "65536"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=_clean_env({}))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["world"] == 2 and d["backend"] == "gloo"
    assert {"allreduce_65536B", "allgather_2967552B", "p2p_64MB_0to1"} <= set(d)
    assert all(v["s"] > 0 for k, v in d.items() if isinstance(v, dict))
