"""Data-parallel parity on 2+ GPUs (skipped on a 1-GPU box): tools/dist_parity.py under
torchrun -- N NCCL ranks on B/N sequences each against one GPU on the whole batch, for both
gradient exchanges (NCCL allreduce + Adam; the fused NVLink peer-memory reduce-scatter +
Adam + all-gather, in push mode -- shards delivered by the backward's epilogues -- and pull
mode; push must equal pull bit for bit).  Tolerance: theta, m and v normwise 1e-5 (fp32
path; only the sum order differs) and 2e-2 (bf16 path) against one GPU, the update 1e-4 / 2e-2
(it is a difference of fp32 thetas: one ulp of theta is ~1e-4 of the update); after step 1
also against the oracle on the whole batch (averaged gradient, m, and the update where the
gradient sign is resolved): 1e-4 (fp32) / 2e-2 (bf16); replicas bit-identical after the
exchange.  The world 2/4/8 arithmetic of the fused kernel is also checked on ONE GPU against
the oracle in test_gpu_dp_emul.py."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs")
@pytest.mark.parametrize("dp", ["fused", "fused-push", "allreduce"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_dp_two_ranks(dp, precision):
    port = 29600 + ["fused", "fused-push", "allreduce"].index(dp) * 10 + (precision == "bf16")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "dist_parity.py"), "--precision", precision, "--dp", dp,
           "--steps", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    res = next(x for x in lines if "theta_err" in x)
    rep = next(x for x in lines if "replicas_identical" in x)
    tol = 1e-5 if precision == "fp32" else 2e-2
    assert res["ok"], json.dumps(res)
    for k in ("theta_err", "m_err", "v_err"):                    # vs one GPU, whole batch
        assert res[k] < tol, (k, res)
    otol = 1e-4 if precision == "fp32" else 2e-2                  # vs the oracle (step 1)
    # the update vs one GPU is a difference of fp32 thetas (one ulp ~ 1e-4 of the update)
    assert res["update_err"] < otol, res
    for k in ("oracle_m_err", "oracle_update_err", "oracle_grad_err"):
        assert res.get(k, 0.0) < otol, (k, res)
    assert res["oracle_firm_frac"] > (0.9 if precision == "fp32" else 0.8), res
    assert rep["replicas_identical"]
    if dp == "fused-push" and precision == "bf16":   # push ran: it must equal pull bitwise
        assert next(x for x in lines if "push_equals_pull" in x)["push_equals_pull"]
