"""Expert-parallel layer, world size 2 over gloo on CPU: the EP
forward (dispatch all-to-all -> local experts -> combine all-to-all) must give
bit-identical outputs to the single-process composed oracle. The local expert
compute here is the CPU oracle (test infrastructure); on B200 boxes it is the
CUDA CompressedMoELayer, with NCCL as the backend."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _make_experts(E, d_model, d_ff, odic):
    from oracle import qmoe_oracle as O

    experts = []
    for e in range(E):
        pair = []
        for m, (rows, cols) in enumerate(((d_ff, d_model), (d_model, d_ff))):
            rng = np.random.default_rng(np.random.SeedSequence([3, e, m]))
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            mm = O.make_grid_bits(w)
            cw, ro = O.encode_codes(O.rtn_codes(w, mm), odic)
            pair.append((rows, cols, cw, ro, mm))
        experts.append(tuple(pair))
    return experts


def _worker(rank, world, port, E, T, out_q, drop=False):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import qmoe_oracle as O
    from paper_2310_16795_b200.ep import ExpertParallelMoE, shard_experts

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    odic = O.OracleDictionary(0.885, O.generate_decode_words(0.885))
    d_model, d_ff = 32, 96
    experts = _make_experts(E, d_model, d_ff, odic)
    mine = [experts[e] for e in shard_experts(E, world, rank)]

    def local_fn(x_recv, local_ids):
        xr = x_recv.numpy()
        ids = local_ids.numpy()
        return torch.from_numpy(O.moe_layer(xr, ids, mine, odic)) if len(ids) else torch.zeros((0, d_model))

    ep = ExpertParallelMoE(E, local_fn)
    rng = np.random.default_rng(100 + rank)
    x = O.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    assign = O.router_argmax(x, E, seed=0)
    if drop:  # tokens without an expert (ids outside [0, E)): zero rows
        assign[::3] = -1
        assign[1::5] = E
    y = ep.forward(torch.from_numpy(x), torch.from_numpy(assign))
    y_ref = O.moe_layer(x, assign, experts, odic)
    out_q.put((rank, bool(np.array_equal(y.numpy(), y_ref)), ep.last_split))
    dist.destroy_process_group()


@pytest.mark.parametrize("T,drop", [(5, False), (16, False), (16, True)])
def test_ep_world2_matches_single_process(T, drop):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 4, T, q, drop)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    # the two ranks exchanged something in both directions at least once
    splits = {r: s for r, _, s in res}
    if not drop:
        assert int(sum(splits[0][0])) == T and int(sum(splits[1][0])) == T
