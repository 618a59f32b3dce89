"""Failures are loud: every device-detected failure of a step reaches the caller as
MP_ERR_DEVICE (status 7), like every error of the reference ABI (capi.cpp:54-70).

Forced conditions (one per host-mapped error word, fsep_types.cuh ErrWord):
  * receive-buffer overflow  -- max_recv_rows too small for the routed segments;
  * restore readiness timeout -- a copy-engine readiness flag is never written
    (test hook), the gate-up GEMM's producer gives up after FSEP_SPIN_TIMEOUT_MS;
  * peer barrier timeout      -- an emulated rank enters a barrier alone;
  * memory guard overrun      -- a byte past the end of an internal buffer.
Each is reported by mp_fsep_layer_check and by the next forward; the words are
cleared once reported, and a clean step afterwards succeeds."""
import numpy as np
import pytest
import torch

from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200._lib import MoeplanError
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec
from test_gpu_layer import make_problem

pytestmark = pytest.mark.gpu
MP_ERR_DEVICE = 7


def _layer(N, E, K, H, F, T, C, **kw):
    pb = make_problem(N, E, K, H, F, T, 1.2, seed=1)
    layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True, **kw))
    for e in range(E):
        layer.load_expert(e, pb["w1"][e].cuda().contiguous(), pb["w3"][e].cuda().contiguous(),
                          pb["w2"][e].cuda().contiguous())
    layer.load_router(pb["wg"].cuda())
    layer.set_layout(PL.even_replication_layout(N, E, C))
    x = torch.cat(pb["xs"]).cuda()
    io = dict(x=x, bias=torch.from_numpy(np.concatenate(pb["biases"])).cuda(), dy=torch.cat(pb["dys"]).cuda(),
              y=torch.empty_like(x), dx=torch.empty_like(x), T=T)
    return layer, io


def _step(layer, io):
    layer.forward(io["x"], io["bias"], io["T"], io["y"])
    layer.backward(io["dy"], io["dx"])


def _expect_device_error(layer, bit, text):
    with pytest.raises(MoeplanError) as ei:
        layer.check()
    assert ei.value.status == MP_ERR_DEVICE
    assert text in str(ei.value)
    assert layer.last_error_bits == 1 << bit
    assert layer.check() == 0  # reported once, then cleared


def test_receive_overflow_is_reported():
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 256, 2
    layer, io = _layer(N, E, K, H, F, T, C, max_recv_rows=128)
    layer.forward(io["x"], io["bias"], io["T"], io["y"])
    _expect_device_error(layer, 0, "receive buffer overflow")
    assert layer.read("status", 0).view(np.int32)[0] == 1 or any(
        layer.read("status", v).view(np.int32)[0] == 1 for v in range(N))
    layer.close()


def test_overflow_reported_by_next_call():
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 256, 2
    layer, io = _layer(N, E, K, H, F, T, C, max_recv_rows=128)
    layer.forward(io["x"], io["bias"], io["T"], io["y"])
    torch.cuda.synchronize()
    with pytest.raises(MoeplanError) as ei:  # the step's own backward already sees it
        layer.backward(io["dy"], io["dx"])
    assert ei.value.status == MP_ERR_DEVICE
    assert layer.check() == 0  # reported once
    layer.close()


@pytest.mark.parametrize("comm", ["ce", "sm"])
def test_restore_readiness_timeout_is_reported(monkeypatch, comm):
    monkeypatch.setenv("FSEP_SPIN_TIMEOUT_MS", "200")
    if comm == "sm":
        monkeypatch.setenv("FSEP_COMM", "sm")
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 256, 4
    layer, io = _layer(N, E, K, H, F, T, C, copy_engine=True)
    _step(layer, io)
    assert layer.check() == 0
    layer.debug_inject("drop_restore_flag")
    _step(layer, io)
    _expect_device_error(layer, 2, "readiness flag timeout")
    _step(layer, io)  # the next restore epoch writes every flag again
    assert layer.check() == 0
    layer.close()


def test_peer_barrier_timeout_is_reported(monkeypatch):
    monkeypatch.setenv("FSEP_SPIN_TIMEOUT_MS", "100")
    N, E, K, H, F, T, C = 2, 8, 2, 256, 256, 128, 4
    layer, io = _layer(N, E, K, H, F, T, C)
    layer.debug_inject("barrier_timeout")
    _expect_device_error(layer, 1, "peer barrier timed out")
    _step(layer, io)
    assert layer.check() == 0
    layer.close()


def test_memory_guard_overrun_is_reported():
    """Every internal buffer is followed by a guard pattern checked on the device by
    mp_fsep_layer_check (the memcheck stand-in on this pool): a one-byte overrun past
    a buffer fails loudly and names the buffer; clean steps leave every guard intact."""
    N, E, K, H, F, T, C = 4, 8, 2, 256, 256, 256, 3
    layer, io = _layer(N, E, K, H, F, T, C, copy_engine=True)
    for _ in range(2):
        _step(layer, io)
    assert layer.check() == 0
    layer.debug_inject("overwrite_guard")
    with pytest.raises(MoeplanError) as ei:
        layer.check()
    assert ei.value.status == MP_ERR_DEVICE and "x_rows" in str(ei.value)
    assert layer.last_error_bits == 1 << 3
    layer.close()
