"""GPU router: qmoe_route vs the reference's RouterSim
(pipeline.py:164-182) and the gated (combine-scaled) fused step."""

import math

import numpy as np
import pytest

from conftest import bf16_ulp_diff

pytestmark = pytest.mark.gpu

q = pytest.importorskip("paper_2310_16795_b200")
torch = pytest.importorskip("torch")
from oracle import qmoe_oracle as O  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)


def _tokens(T, d, seed, bf16):
    x = np.random.default_rng(seed).normal(size=(T, d)).astype(np.float32)
    return q.bf16_round(x) if bf16 else x


@pytest.mark.parametrize("T,d,E,bf16", [(1, 768, 128, True), (64, 768, 128, True), (200, 96, 8, False),
                                        (33, 2080, 2048, True), (0, 64, 8, False)])
def test_hash_rule_is_bit_exact(T, d, E, bf16):
    sim = q.RouterSim(E, rule="hash", seed=3)
    x = _tokens(T, d, T + d, bf16)
    xd = torch.from_numpy(x).cuda()
    if bf16:
        xd = xd.to(torch.bfloat16)
    ids, gate = q.DeviceRouter(sim, d)(xd, gated=True)
    assert np.array_equal(ids.cpu().numpy(), sim.assign(x))
    assert np.all(gate.cpu().numpy() == 1.0)


@pytest.mark.parametrize("T,d,E,skew", [(1, 768, 128, 0.0), (64, 768, 128, 0.0), (256, 768, 128, 0.5),
                                        (40, 2080, 2048, 0.0), (300, 32, 3, 0.0)])
def test_argmax_rule_matches_routersim(T, d, E, skew):
    sim = q.RouterSim(E, rule="argmax", seed=1, skew=skew)
    x = _tokens(T, d, T * 7 + d, True)
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    ids, gate = q.DeviceRouter(sim, d)(xd, gated=True)
    ids, gate = ids.cpu().numpy(), gate.cpu().numpy()
    want = sim.assign(x)
    scores = x.astype(np.float64) @ sim.projection(d) + sim.bias(d)[None, :]
    srt = np.sort(scores, axis=1)
    gap = srt[:, -1] - srt[:, -2] if E > 1 else np.full(T, np.inf)
    near_tie = gap <= 1e-9 * np.abs(srt[:, -1]).clip(min=1.0)
    assert np.all((ids == want) | near_tie), np.flatnonzero((ids != want) & ~near_tie)
    p = np.exp(scores - scores.max(axis=1, keepdims=True))
    p_top = (p / p.sum(axis=1, keepdims=True))[np.arange(T), want]
    np.testing.assert_allclose(gate, p_top.astype(np.float32), rtol=1e-6, atol=1e-30)


def test_argmax_ties_pick_lowest_index():
    # x = 0 gives all-zero scores: np.argmax -> expert 0
    sim = q.RouterSim(16, rule="argmax", seed=0)
    xd = torch.zeros((5, 64), device="cuda")
    ids, gate = q.DeviceRouter(sim, 64)(xd, gated=True)
    assert np.array_equal(ids.cpu().numpy(), sim.assign(np.zeros((5, 64), np.float32)))
    np.testing.assert_allclose(gate.cpu().numpy(), 1.0 / 16, rtol=1e-7)


def test_routed_gated_step_matches_oracle(dic, odic):
    rng = np.random.default_rng(11)
    E, d_model, d_ff, T = 8, 128, 384, 48
    wi, wo, host = [], [], []
    for e in range(E):
        pair = []
        for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            c = q.encode(q.rtn_quantize(w, q.make_grid(w)), dic)
            lst.append(c.to_device(dic))
            pair.append((rows, cols, c.codewords, c.row_off, c.row_minmax))
        host.append(tuple(pair))
    layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=T)
    sim = q.RouterSim(E, rule="argmax", seed=2)
    router = q.DeviceRouter(sim, d_model)
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    y0, a0, g0 = layer.forward_routed(xd, router)
    y1, a1, g1 = layer.forward_routed(xd, router, gated=True)
    assign = a0.cpu().numpy()
    assert np.array_equal(assign, a1.cpu().numpy())
    assert g0 is None
    y_ref = O.moe_layer(x, assign, host, odic)
    d = bf16_ulp_diff(y0.cpu().numpy(), y_ref)
    assert d.max() <= 2 and np.mean(d == 0) >= 0.99
    # gated rows: exactly gate[t] * ungated row (one f32 multiply)
    gate = g1.cpu().numpy()
    assert np.array_equal(y1.cpu().numpy(), (y0.cpu().numpy() * gate[:, None]).astype(np.float32))
    assert np.all((gate > 0) & (gate <= 1))
    assert math.isfinite(float(gate.sum()))


def test_device_router_matches_reference_golden(golden):
    """qmoe_route against RouterSim.assign outputs of the reference itself
    (tests/golden/routing.npz, made by tests/golden/make_golden.py)."""
    g = golden("routing.npz")
    for i in range(int(g["n"])):
        E, d, T, seed = (int(v) for v in g[f"c{i}_meta"])
        rule, skew = str(g[f"c{i}_rule"]), float(g[f"c{i}_skew"])
        xbits = torch.from_numpy(g[f"c{i}_xbits"].view(np.int16).copy()).cuda()
        ids, _ = q.DeviceRouter(q.RouterSim(E, rule=rule, seed=seed, skew=skew), d)(xbits.view(torch.bfloat16))
        assert np.array_equal(ids.cpu().numpy(), g[f"c{i}_assign"]), (rule, E, d)
