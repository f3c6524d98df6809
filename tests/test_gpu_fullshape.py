"""GPU parity at the BASELINE configs' full layer shapes:
the timed paths themselves — the fused step on a Switch-base-128 layer (128
experts, 768/3072, the step's 32K hot-table cap, multi-window walks), the
decode-then-MMA passes on a Switch-large-128 layer (1024/4096), the fused step
on a c2048-shaped layer (2080/6144, 256 experts) — against the composed CPU
oracle (moepack.codec.fused_matvec restated) on the same device streams, plus
GPU RTN and the GPU encoder against the oracle's at full matrix sizes.

Bars: MoE outputs <= 2 bf16 ulp, >= 99% identical (compared on up to 16
sampled tokens per step: the oracle costs ~30-150 ms per token); RTN codes,
grids and codeword streams bit-exact."""

import numpy as np
import pytest

from conftest import bf16_ulp_diff

pytestmark = pytest.mark.gpu

q = pytest.importorskip("paper_2310_16795_b200")
torch = pytest.importorskip("torch")
from oracle import qmoe_oracle as O  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2310_16795_b200.synth import build_layer, seeded_weights  # noqa: E402


def host_streams(m):
    """(rows, cols, codewords in dictionary order, row_off, (rows, 2) bf16
    min/max) of a device matrix — what the reference codec holds (undoes the
    layer's kernel-private frequency codebook)."""
    cw = m.cw.cpu().numpy().view(np.uint16)
    if m.codebook is not None:
        cw = m.codebook.order[cw]
    return (m.rows, m.cols, cw, m.row_off.cpu().numpy(),
            m.row_minmax.cpu().numpy().view(np.uint16).reshape(m.rows, 2))


def oracle_tokens(layer, x, assign, toks, odic):
    """Composed oracle outputs of the sampled tokens (per token: wi matvec ->
    ReLU -> wo matvec, codec.py:209-244 per matvec)."""
    host = {}
    y = np.zeros((len(toks), layer.d_model), np.float32)
    for k, t in enumerate(toks):
        e = int(assign[t])
        if not 0 <= e < layer.E:
            continue
        if e not in host:
            host[e] = (host_streams(layer.wi[e]), host_streams(layer.wo[e]))
        wi, wo = host[e]
        h = O.fused_matvec(*wi[:2], *wi[2:], odic.hash64, x[t], odic, workers=8)
        y[k] = O.fused_matvec(*wo[:2], *wo[2:], odic.hash64, np.maximum(h, 0.0), odic, workers=8)
    return y


def check(y_gpu, y_ref):
    d = bf16_ulp_diff(y_gpu, y_ref)
    assert d.max() <= 2, f"max {d.max()} bf16 ulp"
    assert np.mean(d == 0) >= 0.99, f"only {np.mean(d == 0):.4f} identical"


@pytest.fixture(scope="module")
def base_layer(dic):
    return build_layer(128, 768, 3072, seed=21, dic=dic, max_tokens=64)


@pytest.mark.parametrize("T", [1, 8, 64])
def test_switch_base_128_fused_step_vs_oracle(dic, odic, base_layer, T):
    layer = base_layer
    assert layer.fused and not layer.use_dense(T)
    rng = np.random.default_rng(1000 + T)
    x = q.bf16_round(rng.normal(size=(T, 768)).astype(np.float32))
    assign = q.RouterSim(128, rule="argmax", seed=0).assign(x)
    y = layer.forward_device(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(assign).cuda())
    toks = np.sort(rng.choice(T, size=min(T, 16), replace=False))
    check(y.cpu().numpy()[toks], oracle_tokens(layer, x, assign, toks, odic))


def test_switch_base_128_host_api_vs_oracle(dic, odic, base_layer):
    """The drop-in host API (numpy in / out, the e2e path) on the full layer."""
    rng = np.random.default_rng(77)
    x = q.bf16_round(rng.normal(size=(64, 768)).astype(np.float32))
    assign = q.RouterSim(128, rule="argmax", seed=0).assign(x)
    y = base_layer.forward(x, assign)
    toks = np.arange(0, 64, 4)
    check(y[toks], oracle_tokens(base_layer, x, assign, toks, odic))


def test_switch_large_128_dense_pass_vs_oracle(dic, odic):
    layer = build_layer(128, 1024, 4096, seed=22, dic=dic, max_tokens=1024)
    layer.dense_mode = "always"
    T = 1024
    rng = np.random.default_rng(5)
    x = q.bf16_round(rng.normal(size=(T, 1024)).astype(np.float32))
    assign = q.RouterSim(128, rule="argmax", seed=0).assign(x)
    assert layer.use_dense(T)
    y = layer.forward_device(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(assign).cuda())
    toks = np.sort(rng.choice(T, size=16, replace=False))
    check(y.cpu().numpy()[toks], oracle_tokens(layer, x, assign, toks, odic))
    # the streaming step computes the same outputs (<= 2 ulp apart)
    layer.dense_mode = "never"
    y2 = layer.forward_device(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(assign).cuda())
    assert bf16_ulp_diff(y.cpu().numpy(), y2.cpu().numpy()).max() <= 2


def test_c2048_shaped_layer_fused_step_vs_oracle(dic, odic):
    E, d_model, d_ff, T = 256, 2080, 6144, 8
    layer = build_layer(E, d_model, d_ff, seed=23, dic=dic, max_tokens=T)
    rng = np.random.default_rng(6)
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    assign = q.RouterSim(E, rule="argmax", seed=0).assign(x)
    assign[1] = assign[0]  # one expert with two tokens (a 2-token run)
    y = layer.forward_device(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(assign).cuda())
    toks = np.arange(T)
    check(y.cpu().numpy(), oracle_tokens(layer, x, assign, toks, odic))


@pytest.mark.parametrize("rows,cols", [(768, 3072), (2080, 6144)])
def test_gpu_rtn_and_encode_full_size_vs_oracle(dic, odic, rows, cols):
    """GPU make_grid + RTN (quantize.py:91-126, 219-235) and the GPU encoder
    (codec.py:126-155) on the survey's seeded weights: bit-exact."""
    from paper_2310_16795_b200.codec import encode_device
    from paper_2310_16795_b200.quantize import rtn_quantize_device

    w = seeded_weights(0, 0, 3, 1, rows, cols)
    codes, mm = rtn_quantize_device(torch.from_numpy(w).cuda())
    mm_ref = O.make_grid_bits(w)
    codes_ref = O.rtn_codes(w, mm_ref)
    assert np.array_equal(mm.cpu().numpy().view(np.uint16).reshape(rows, 2), mm_ref)
    assert np.array_equal(codes.cpu().numpy(), codes_ref)
    dm = encode_device(codes, mm, dic)
    cw_ref, ro_ref = O.encode_codes(codes_ref, odic)
    assert np.array_equal(dm.row_off.cpu().numpy(), ro_ref)
    assert np.array_equal(dm.cw.cpu().numpy().view(np.uint16), cw_ref)
