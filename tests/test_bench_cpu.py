"""bench.py's launch contract on CPU (no GPU needed): `--gpus N` without torchrun starts N ranks (it re-launches
itself under torch.distributed.run), every rank joins, and rank 0 alone prints one JSON line.  The reference arm
(the oracle) runs on the host, so the multi-rank launch path is exercised here."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_gpus2_starts_two_ranks():
    line = _run(["--gpus", "2", "--impl", "reference", "--workload", "config1", "--steps", "1", "--warmup", "0"])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["ranks_started"] == 2
    assert line["config"]["parallelism"].startswith("dp2")


def test_bench_reference_arm_single_rank():
    line = _run(["--impl", "reference", "--workload", "config1", "--steps", "1", "--warmup", "0"])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
