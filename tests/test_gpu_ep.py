"""Expert-parallel exchange kernels on the GPU: fixed-slot
dispatch (qmoe_ep_slots) and row moves (qmoe_ep_rows) against a numpy
restatement, and the EP layer at world size 1 over NCCL against the local
layer (bit-identical)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

q = pytest.importorskip("paper_2310_16795_b200")
torch = pytest.importorskip("torch")

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2310_16795_b200 import _lib  # noqa: E402


def _slots_ref(assign, E, W):
    T = len(assign)
    per = E // W
    slot = np.full(T, -1, np.int64)
    ids = np.full(W * T, -1, np.int64)
    cnt = np.zeros(W, np.int64)
    for t, a in enumerate(assign):
        if 0 <= a < E:
            d = a // per
            slot[t] = d * T + cnt[d]
            ids[slot[t]] = a - d * per
            cnt[d] += 1
    return slot, ids, cnt


@pytest.mark.parametrize("T,E,W", [(1, 8, 1), (64, 128, 4), (300, 2048, 8), (2500, 64, 64), (37, 6, 3)])
def test_ep_slots_match_reference(T, E, W):
    rng = np.random.default_rng(T + E + W)
    a = rng.integers(-2, E + 2, size=T).astype(np.int32)
    ad = torch.from_numpy(a).cuda()
    slot = torch.empty(T, dtype=torch.int32, device="cuda")
    ids = torch.empty(W * T, dtype=torch.int32, device="cuda")
    cnt = torch.empty(W, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib.qmoe_ep_slots(_lib.ptr(ad), T, E, W, _lib.ptr(slot), _lib.ptr(ids), _lib.ptr(cnt),
                                      _lib.stream_ptr()))
    rs, ri, rc = _slots_ref(a, E, W)
    assert np.array_equal(slot.cpu().numpy(), rs)
    assert np.array_equal(ids.cpu().numpy(), ri)
    assert np.array_equal(cnt.cpu().numpy(), rc)
    # rows: scatter then gather back is the identity on valid tokens, zero elsewhere
    x = torch.randn(T, 96, device="cuda")
    xs = torch.full((W * T, 96), 7.0, device="cuda")
    _lib.check(_lib.lib.qmoe_ep_rows(_lib.ptr(x), _lib.ptr(xs), T, 96 * 4, _lib.ptr(slot), 1, _lib.stream_ptr()))
    back = torch.empty_like(x)
    _lib.check(_lib.lib.qmoe_ep_rows(_lib.ptr(xs), _lib.ptr(back), T, 96 * 4, _lib.ptr(slot), 0, _lib.stream_ptr()))
    ok = torch.from_numpy(rs >= 0).cuda()
    assert torch.equal(back[ok], x[ok])
    assert torch.all(back[~ok] == 0)


def test_ep_layer_world1_nccl_matches_local(dic):
    import torch.distributed as dist

    from paper_2310_16795_b200.ep import ExpertParallelMoE

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(9)
        E, d_model, d_ff, T = 8, 128, 256, 40
        wi, wo = [], []
        for e in range(E):
            for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
                w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
                lst.append(q.encode(q.rtn_quantize(w, q.make_grid(w)), dic).to_device(dic))
        layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=T)
        x = torch.from_numpy(q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))).cuda()
        a_np = rng.integers(-1, E, size=T).astype(np.int32)
        a = torch.from_numpy(a_np).cuda()
        ep = ExpertParallelMoE(E, lambda xr, ir: layer.forward_device(xr, ir))
        y_ep = ep.forward(x, a)
        y_loc = layer.forward_device(x, a)
        ok = torch.from_numpy(a_np >= 0).cuda()
        assert torch.equal(y_ep[ok], y_loc[ok])
        assert torch.all(y_ep[~ok] == 0)
    finally:
        dist.destroy_process_group()
