"""CPU checks of the C-ABI library: it loads, exports every symbol include/ppo5.h declares,
and rejects bad arguments on the host without touching a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ppo5.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1912_06680_b200 import _lib
    return _lib


def test_header_declares_the_hot_path():
    names = _declared()
    for n in ("ppo_gae", "lstm_bptt_fwd", "lstm_bptt_bwd", "ppo_loss_grad", "grad_allreduce",
              "adam_step", "lstm_ws_bytes", "ppo_comm_init"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(so, n)]
    assert not missing, missing
    assert set(_declared()) == set(lib.EXPORTED)


def test_host_side_errors(lib):
    d = lib.make_dims(4032, 4096, 16, (30, 4, 189, 189, 81, 81, 81))
    lay = lib.param_layout(d)
    assert lay.Kx == 4032 + 4096 + 64 and lay.Ko == 4096 + 64 and lay.A == 656
    assert lay.n_total == 4 * 4096 * lay.Kx + 656 * lay.Ko
    bad = lib.make_dims(4000, 4096, 16, (30,))
    with pytest.raises(lib.PPOError) as e:
        lib.param_layout(bad)
    assert e.value.code == lib.PPO_E_SHAPE
    assert "multiples of 64" in lib.last_error()
    with pytest.raises(lib.PPOError):
        lib.ws_bytes(d, 0)
    # workspace size matches the documented layout (bf16 activations)
    B = 40
    n = lib.ws_bytes(d, B)
    assert n >= (17 * B * lay.Kx * 2 + 16 * B * 4 * 4096 * 2 + 17 * B * 4096 * 4 + B * 4096 * 4)
    assert "sm_100a" in lib.version()


def test_null_pointers_rejected(lib):
    d = lib.make_dims(256, 128, 16, (30, 4, 189, 189, 81, 81, 81))
    rc = lib._lib.adam_step(None, None, None, None, None, 10, 1, 1e-3, 0.9, 0.999, 1e-8, 5.0, None)
    assert rc == lib.PPO_E_ARG
    rc = lib._lib.ppo_gae(None, None, None, 2, 256, 0.99, 0.95, 0, None, None, None, 0, None)
    assert rc == lib.PPO_E_ARG
    rc = lib._lib.ppo_gae(None, None, None, 0, 256, 0.99, 0.95, 0, None, None, None, 0, None)
    assert rc == lib.PPO_OK  # empty input is a no-op
    assert lib.gae_scratch_bytes(4, 256) == 0
    assert lib.gae_scratch_bytes(1, 10 ** 6) >= 16 * (10 ** 6 // 4096)
    assert lib.gae_scratch_bytes(20000, 20000) == 0  # enough streams: warp per stream


def test_next_rows_host_checks(lib):
    """Host-side argument checks of the §8(f) calls (no device needed)."""
    hs = (30, 4, 189, 189, 81, 81, 81)
    # aux heads: sizes bounded; A counts them; bad trunk weight rejected
    d = lib.make_dims(256, 128, 16, hs, lib.PPO_PREC_BF16, (1, 5, 18), 0.01)
    assert lib.param_layout(d).A == 656 + 24
    with pytest.raises(lib.PPOError) as e:
        lib.param_layout(lib.make_dims(256, 128, 16, hs, lib.PPO_PREC_BF16, (2, 5, 18), 0.01))
    assert e.value.code == lib.PPO_E_SHAPE
    with pytest.raises(lib.PPOError) as e:
        lib.param_layout(lib.make_dims(256, 128, 16, hs, lib.PPO_PREC_BF16, (1, 33, 0), 0.01))
    assert e.value.code == lib.PPO_E_SHAPE
    with pytest.raises(lib.PPOError) as e:
        lib.param_layout(lib.make_dims(256, 128, 16, hs, lib.PPO_PREC_BF16, (1, 5, 18), -1.0))
    assert e.value.code == lib.PPO_E_ARG
    # inference workspace / weights sizes are positive and grow with B
    dims = lib.make_dims(256, 128, 1, hs)
    assert 0 < lib.infer_ws_bytes(dims, 1) < lib.infer_ws_bytes(dims, 64)
    assert lib.infer_weights_bytes(dims) >= 2 * (4 * 128 * (256 + 128 + 64) + 656 * (128 + 64))
    # the inference step needs the bf16 path and non-NULL buffers
    rc = lib._lib.ppo_infer_step(ctypes.byref(lib.make_dims(256, 128, 1, hs, lib.PPO_PREC_FP32)),
                                 None, None, None, None, None, None, 0, 0, 60, None, 0, None, None,
                                 None, None, None, None)
    assert rc == lib.PPO_E_ARG
    rc = lib._lib.ppo_infer_step(ctypes.byref(dims), None, None, None, None, None, None, 0, 0, 60,
                                 None, 0, None, None, None, None, None, None)
    assert rc == lib.PPO_E_ARG
    # aux labels: L must be a multiple of seq_T
    rc = lib._lib.ppo_aux_labels(ctypes.byref(d), 2, 250, None, None, None, None, None,
                                 ctypes.c_float(0.999), 16, None, None)
    assert rc == lib.PPO_E_SHAPE
    # reward pipeline: scratch size and config checks
    assert lib.reward_gae_scratch_bytes() > 0
    # streamed x: slice index checked
    rc = lib._lib.ppo_copy_x_slice(ctypes.byref(lib.make_dims(256, 128, 16, hs)), 8, 16, None, 256,
                                   None, 0, None)
    assert rc == lib.PPO_E_SHAPE


def test_dp_fused_host_checks(lib):
    """The fused a9+a10 exchange (ppo_dp_*): shard arithmetic and host-side argument checks."""
    for n in (1, 63, 64, 1000, 135_917_728, 135_917_729):
        for world in (1, 2, 3, 4, 8):
            s = lib.dp_shard(n, world)
            assert s % 64 == 0 and world * s >= n and s - -(-n // world) < 64, (n, world, s)
    assert lib.dp_shard(10, 0) == 0
    assert lib._lib.ppo_dp_attach(None, None, None, None, 10) == lib.PPO_E_ARG
    assert lib._lib.ppo_dp_adam_step(None, None, None, 1, 1e-3, 0.9, 0.999, 1e-8, 5.0, 0,
                                     None) == lib.PPO_E_ARG
    hs = (30, 4, 189, 189, 81, 81, 81)
    d = lib.make_dims(256, 128, 16, hs)
    assert lib._lib.lstm_bptt_bwd_dp(ctypes.byref(d), None, None, 0, None, 32, None, None,
                                     None) == lib.PPO_E_ARG
    assert lib._lib.ppo_dp_allgather(None, None, None) == lib.PPO_E_ARG
    assert "comm is NULL" in lib.last_error()


def test_empty_and_degenerate_sizes(lib):
    """Empty elementwise inputs are no-ops (before any pointer check); B = 0 is rejected by
    the LSTM and loss calls (include/ppo5.h, conventions) -- all decided on the host."""
    assert lib._lib.adam_step(None, None, None, None, None, 0, 1, 1e-3, 0.9, 0.999, 1e-8, 5.0,
                              None) == lib.PPO_OK
    assert lib._lib.ppo_gae(None, None, None, 3, 0, 0.99, 0.95, 0, None, None, None, 0,
                            None) == lib.PPO_OK
    assert lib._lib.ppo_gae(None, None, None, -1, 4, 0.99, 0.95, 0, None, None, None, 0,
                            None) == lib.PPO_E_SHAPE
    assert lib.gae_scratch_bytes(0, 10 ** 6) == 0
    d = lib.make_dims(256, 128, 16, (30, 4, 189, 189, 81, 81, 81))
    rc = lib._lib.lstm_bptt_bwd(ctypes.byref(d), None, None, 0, None, 0, None, None)
    assert rc == lib.PPO_E_SHAPE and "B must be >= 1" in lib.last_error()
    rc = lib._lib.ppo_loss_grad(ctypes.byref(d), None, None, None, None, None, None, None, None,
                                None, 0, None, None, None, None, None)
    assert rc == lib.PPO_E_SHAPE and "B must be >= 1" in lib.last_error()
