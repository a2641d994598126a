"""bench.py's CPU-side contract (no GPU): the reference arm (the oracle timed on the host cores)
prints one JSON line with the keys the driver reads, for the default workload and for the other
arms of the --config / --rt-reading switches."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("args", [["--config", "1"], ["--config", "2", "--steps", "3"],
                                  ["--config", "3", "--steps", "3", "--rt-reading", "literal"]])
def test_reference_arm_json_line(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--warmup", "3"] + args, capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "apply/s"
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "dtype",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    if "--rt-reading" in args:
        assert d["config"]["workload"].endswith("_literal_c3")
    if args[1] == "2":
        assert d["vs_baseline"] is not None


def test_reference_arm_honours_steps_and_matches_gpu_config():
    """The reference arm runs exactly --steps timed applications after --warmup (floor 3, as the
    GPU arm) and prints the config dict the GPU arm builds for the same workload (one helper)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "2", "--steps", "4", "--warmup", "1"], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["steps"] == 4 and d["warmup"] == 3
    sys.path.insert(0, ROOT)
    import bench
    import synth
    from oracle import spaces
    w = synth.CONFIGS[2]
    n_total = spaces.build(w.dim, w.disc, w.p, w.n_el).n_total
    assert d["config"] == bench.workload_config(2, w, n_total, 1)


def test_bench_default_is_config5():
    """The driver's bench line is the largest single-GPU configuration (config 5)."""
    sys.path.insert(0, ROOT)
    import bench
    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = bench.parse()
    finally:
        sys.argv = old
    assert a.config == 5 and a.gpus == 1
    flush, l2 = bench.l2_policy(548753616, 1)
    assert not flush and "no flush" in l2
