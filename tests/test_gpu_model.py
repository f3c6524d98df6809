"""The synthetic compressed model (BASELINE config 5 structure): residual
blocks, routing on the device, one fused launch per block
(qmoe_moe_step_resid), checked layer by layer against the composed CPU oracle
(routing: RouterSim hash, bit-exact; expert FFN: moepack.codec.fused_matvec
restated; residual: bf16(x + y))."""

import numpy as np
import pytest

from conftest import bf16_ulp_diff

pytestmark = pytest.mark.gpu

q = pytest.importorskip("paper_2310_16795_b200")
torch = pytest.importorskip("torch")
from oracle import qmoe_oracle as O  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)


def _layer(dic, rng, E, d_model, d_ff, T):
    wi, wo, host = [], [], []
    for e in range(E):
        pair = []
        for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            c = q.encode(q.rtn_quantize(w, q.make_grid(w)), dic)
            lst.append(c.to_device(dic))
            pair.append((rows, cols, c.codewords, c.row_off, c.row_minmax))
        host.append(tuple(pair))
    return q.CompressedMoELayer(wi, wo, dic, max_tokens=T), host


@pytest.mark.parametrize("T", [1, 12, 70])
def test_model_forward_layer_by_layer_vs_oracle(dic, odic, T):
    rng = np.random.default_rng(60 + T)
    E, d_model, d_ff, L = 5, 96, 224, 3
    built = [_layer(dic, rng, E, d_model, d_ff, T) for _ in range(L)]
    sims = [q.RouterSim(E, rule="hash", seed=10 + l) for l in range(L)]
    routers = [q.DeviceRouter(s, d_model) for s in sims]
    model = q.CompressedMoEModel([b[0] for b in built], routers)
    x0 = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    out, trace = model.forward_device(torch.from_numpy(x0).cuda().to(torch.bfloat16), keep=True)
    inputs = [t[0].float().cpu().numpy() for t in trace] + [out.float().cpu().numpy()]
    assert np.array_equal(inputs[0], x0)
    for l in range(L):
        x = inputs[l]
        ids = trace[l][1].cpu().numpy()
        assert np.array_equal(ids, sims[l].assign(x)), "device routing differs from RouterSim"
        y = O.moe_layer(x, ids, built[l][1], odic)
        want = O.bf16_round(x + y)  # residual add in f32, one bf16 rounding
        d = bf16_ulp_diff(inputs[l + 1], want)
        rel = np.linalg.norm(inputs[l + 1] - want) / max(np.linalg.norm(want), 1e-30)
        assert np.mean(d == 0) >= 0.99 and rel <= 1e-2, (l, d.max(), np.mean(d == 0), rel)


def test_model_forward_is_graph_capturable_and_gated(dic):
    """The gated block equals the routed step plus a residual add; the whole
    forward replays from a CUDA graph."""
    rng = np.random.default_rng(8)
    E, d_model, d_ff, L, T = 4, 64, 192, 2, 16
    built = [_layer(dic, rng, E, d_model, d_ff, T) for _ in range(L)]
    routers = [q.DeviceRouter(q.RouterSim(E, rule="argmax", seed=l), d_model) for l in range(L)]
    model = q.CompressedMoEModel([b[0] for b in built], routers, gated=True)
    x = torch.from_numpy(q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))).cuda().to(torch.bfloat16)
    ref = x
    for lay, r in zip(model.layers, routers):
        y, _, _ = lay.forward_routed(ref, r, gated=True)
        ref = (ref.float() + y).to(torch.bfloat16)  # RNE of the f32 sum, as the fused store
    got = model.forward_device(x)
    assert torch.equal(got, ref)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        model.forward_device(x)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = model.forward_device(x)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
