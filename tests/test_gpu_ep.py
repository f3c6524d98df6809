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


def _slots_ref(assign, E, W, C):
    T = len(assign)
    per = E // W
    slot = np.full(T, -1, np.int64)
    ids = np.full(W * C, -1, np.int64)
    cnt = np.zeros(W, np.int64)
    for t, a in enumerate(assign):
        if 0 <= a < E:
            d = a // per
            slot[t] = d * C + cnt[d]
            ids[slot[t]] = a - d * per
            cnt[d] += 1
    return slot, ids, cnt


@pytest.mark.parametrize("T,E,W,extra", [(1, 8, 1, 0), (64, 128, 4, 0), (300, 2048, 8, 5), (2500, 64, 64, 0),
                                         (37, 6, 3, 11)])
def test_ep_slots_match_reference(T, E, W, extra):
    C = T + extra  # slots per destination: the layer's capacity (>= T)
    rng = np.random.default_rng(T + E + W)
    a = rng.integers(-2, E + 2, size=T).astype(np.int32)
    ad = torch.from_numpy(a).cuda()
    slot = torch.empty(T, dtype=torch.int32, device="cuda")
    ids = torch.empty(W * C, dtype=torch.int32, device="cuda")
    cnt = torch.empty(W, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib.qmoe_ep_slots(_lib.ptr(ad), T, E, W, C, _lib.ptr(slot), _lib.ptr(ids), _lib.ptr(cnt),
                                      _lib.stream_ptr()))
    rs, ri, rc = _slots_ref(a, E, W, C)
    assert np.array_equal(slot.cpu().numpy(), rs)
    assert np.array_equal(ids.cpu().numpy(), ri)
    assert np.array_equal(cnt.cpu().numpy(), rc)
    # rows: scatter then gather back is the identity on valid tokens, zero elsewhere
    x = torch.randn(T, 96, device="cuda")
    xs = torch.full((W * C, 96), 7.0, device="cuda")
    _lib.check(_lib.lib.qmoe_ep_rows(_lib.ptr(x), _lib.ptr(xs), T, 96 * 4, _lib.ptr(slot), 1, _lib.stream_ptr()))
    back = torch.empty_like(x)
    _lib.check(_lib.lib.qmoe_ep_rows(_lib.ptr(xs), _lib.ptr(back), T, 96 * 4, _lib.ptr(slot), 0, _lib.stream_ptr()))
    ok = torch.from_numpy(rs >= 0).cuda()
    assert torch.equal(back[ok], x[ok])
    assert torch.all(back[~ok] == 0)
    # bf16 combine gather: exact widening, zero rows for tokens without an expert
    xb = xs.to(torch.bfloat16)
    yc = torch.full((T, 96), 3.0, device="cuda")
    _lib.check(_lib.lib.qmoe_ep_combine(_lib.ptr(xb), _lib.ptr(yc), T, 96, _lib.ptr(slot), _lib.stream_ptr()))
    assert torch.equal(yc[ok], x[ok].to(torch.bfloat16).float())
    assert torch.all(yc[~ok] == 0)
    with pytest.raises(ValueError):  # capacity below the token count
        _lib.check(_lib.lib.qmoe_ep_slots(_lib.ptr(ad), T, E, W, T - 1, _lib.ptr(slot), _lib.ptr(ids),
                                          _lib.ptr(cnt), _lib.stream_ptr()))


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


def _ep_gpu_worker(rank, world, port, E, T, out_q):
    """One rank of the world-2 CUDA-path test: its block of experts as a
    CompressedMoELayer on cuda:0 (both ranks share the GPU), the device
    dispatch/combine kernels, gloo (host-staged) all-to-alls."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_2310_16795_b200 as qq
    from oracle import qmoe_oracle as O
    from paper_2310_16795_b200.ep import ExpertParallelMoE, shard_experts

    try:
        torch.cuda.set_device(0)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dic = qq.generate_dictionary()
        odic = O.OracleDictionary(0.885, dic.decode_words)
        d_model, d_ff = 128, 384
        host, dev = [], []
        for e in range(E):
            pair, mats = [], []
            for m, (rows, cols) in enumerate(((d_ff, d_model), (d_model, d_ff))):
                rng = np.random.default_rng(np.random.SeedSequence([11, e, m]))
                w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
                c = qq.encode(qq.rtn_quantize(w, qq.make_grid(w)), dic)
                pair.append((rows, cols, c.codewords, c.row_off, c.row_minmax))
                mats.append(c)
            host.append(tuple(pair))
            dev.append(mats)
        mine = list(shard_experts(E, world, rank))
        layer = qq.CompressedMoELayer([dev[e][0].to_device(dic) for e in mine],
                                      [dev[e][1].to_device(dic) for e in mine], dic, max_tokens=world * (T + 3))
        ep = ExpertParallelMoE(E, lambda xr, ir: layer.forward_device(xr, ir), max_tokens=T + 3)
        rng = np.random.default_rng(500 + rank)
        Tr = T - rank  # ranks bring different token counts (<= the capacity)
        x = O.bf16_round(rng.normal(size=(Tr, d_model)).astype(np.float32))
        assign = O.router_argmax(x, E, seed=0)
        assign[::7] = -1  # some tokens without an expert
        y = ep.forward(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(assign).cuda())
        y_ref = O.moe_layer(x, assign, host, odic)
        d = np.abs(y.cpu().numpy().view(np.int32).astype(np.int64) - y_ref.view(np.int32).astype(np.int64)) >> 16
        out_q.put((rank, int(d.max()), float(np.mean(d == 0)), bool(np.all(y.cpu().numpy()[assign < 0] == 0))))
        dist.destroy_process_group()
    except Exception as exc:  # report instead of hanging the parent
        out_q.put((rank, repr(exc), 0.0, False))


def test_ep_world2_cuda_path_vs_oracle():
    """World size 2 on the CUDA path (_forward_device: qmoe_ep_slots /
    qmoe_ep_rows / qmoe_ep_combine around the exchange, the fused local step
    per rank) against the composed CPU oracle; ranks with different token
    counts under one capacity."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_ep_gpu_worker, args=(r, 2, port, 8, 24, qu)) for r in range(2)]
    for p in procs:
        p.start()
    res = [qu.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, maxd, ident, zero_ok in res:
        assert isinstance(maxd, int), (rank, maxd)
        assert maxd <= 2 and ident >= 0.99 and zero_ok, (rank, maxd, ident, zero_ok)
