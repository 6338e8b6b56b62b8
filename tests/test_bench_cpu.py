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


def test_roofline_fields_from_a_synthetic_profile():
    """The roofline block from a per-class profile: L1 bound, algorithmic bytes = evaluations x 600 B
    over the class's time against the measured L1 peak, the ncu-measured hardware fraction of the same kernel, and
    the per-class ncu figures; the FP32 figure beside it."""
    sys.path.insert(0, ROOT)
    import bench
    from types import SimpleNamespace
    wl = bench.WORKLOADS["config2"]
    cfg = SimpleNamespace(loss=2)
    prof = {"field123.L0": {"ms": 1000.0, "launches": 20, "work": 4.0e10},
            "field0.L0": {"ms": 300.0, "launches": 20, "work": 1.0e10},
            "tbar.L0": {"ms": 200.0, "launches": 20, "work": 5.0e9}}
    roof, alu = bench.roofline(prof, wl, cfg, 1)
    assert roof["kernel"] == "pm_field123.L0" and roof["bound"] == "l1" and roof["unit"] == "GB/s"
    assert abs(roof["achieved"] - 4.0e10 * 600 / 1.0 / 1e9) < 1e-6 * roof["achieved"]
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-12
    assert 0.0 < roof["hardware"]["frac"] <= 1.0 and roof["hardware"]["basis"] == "ncu measured"
    assert set(roof["classes"]) >= {"field123.L0", "field0.L0", "tbar.L0"}
    for v in roof["classes"].values():
        assert 0.0 < v["l1_frac_ncu"] <= 1.0
    assert abs(roof["share_of_kernel_time"] - 1000.0 / 1500.0) < 1e-12
    assert alu["bound"] == "alu" and 0.0 < alu["frac"]
