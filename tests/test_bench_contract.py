"""The bench.py JSON contract on CPU: the reference arm (the oracle, the only arm that runs
without a GPU) prints one line with the keys the driver reads, at a tiny shape; the
algorithmic work table covers every kernel class the step launches."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--H", "64",
           "--D", "64", "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=dict(os.environ, OMP_NUM_THREADS="2"))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]


def test_algorithmic_table_covers_the_step():
    sys.path.insert(0, ROOT)
    import bench
    alg = bench.algorithmic(4096, 4032, 16, 38400, 656, 135_900_000)
    for k in ("lstm_fwd_step", "heads_fwd", "lstm_bwd_step", "wgrad_xh", "wgrad_o", "gae",
              "loss", "adam", "pack_state"):
        assert k in alg
    flop = sum(w for kind, w in alg.values() if kind == "flop") - alg["input_grad"][1]
    # F_seq = 2T 4H (2D + 3H) + 6 T H A per sequence; the bench counts the
    # recurrent dh GEMM over the T - 1 steps that have one (1.2% less)
    T, H, D, A, B = 16, 4096, 4032, 656, 38400
    f_seq = 2 * T * 4 * H * (2 * D + 3 * H) + 6 * T * H * A
    exact = f_seq - 2 * 4 * H * H
    assert abs(flop / B - exact) / exact < 1e-9, (flop / B, exact)
