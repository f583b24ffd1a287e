"""bench.py's reference arm (the fp64 oracle on host cores) runs without a GPU: one JSON line with
the contract's keys, the same metric / unit / workload description as our arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, cwd=ROOT,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    sys.path.insert(0, ROOT)
    import bench
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["value"] > 0 and d["higher_is_better"] is True and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("c2 problem (BASELINE configs[1] recipe")
    assert d["config"]["inner_sweeps"] == 20


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (torch.distributed.run on
    127.0.0.1); the self-test mode runs the same barrier / max-over-ranks plumbing over gloo without
    kernels and rank 0 alone prints the line."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--launcher-selftest", "--warmup", "3"],
                         capture_output=True, text=True, cwd=ROOT, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d == {"selftest": True, "n_gpus": 2, "gpus_arg": 2, "max_over_ranks": 2.0}


def test_roofline_byte_and_flop_rules():
    sys.path.insert(0, ROOT)
    import bench
    n = 16384
    # projection 8 m^2 k + 12 n n' = 46.17 GB at c5; per-step B_alg 53.7 GB
    assert bench.proj_alg_bytes(n, n, 20) == 8 * n * n * 20 + 12 * n * n
    assert abs(bench.proj_alg_bytes(n, n, 20) / 1e9 - 46.17) < 0.01
    assert abs(bench.step_alg_bytes(n, n, 20, True) / 1e9 - 53.7) < 0.1
    assert bench.proj_alg_bytes(800, 1000, 3) == 8 * 1000 * 1000 * 3 + 12 * 800 * 1000
    mp = {"bf16_tflops_sustained": 1413.1, "bf16_tflops": 1689.1, "hbm_gbs": 6546.2}
    peak, bound, _ = bench.gemm_peak(mp, "measured", 3)
    assert bound == "tensor" and abs(peak - 1413.1 * 2 / 6) < 1e-9
    assert abs(bench.gemm_peak(mp, "measured", 0)[0] - 1413.1 * 1.1 / 2.25 / 3) < 1e-9
