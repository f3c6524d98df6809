"""GPU parity of the MoE layer (dispatcher + grouped passes) against the
composed reference oracle (<= 2 bf16 ulp per output)."""

import numpy as np
import pytest

from conftest import bf16_ulp_diff

pytestmark = pytest.mark.gpu

q = pytest.importorskip("paper_2310_16795_b200")
torch = pytest.importorskip("torch")
from oracle import qmoe_oracle as O  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)


def layer_from_golden(g, dic):
    E = int(g["E"])
    wi, wo = [], []
    for e in range(E):
        for m, lst in ((0, wi), (1, wo)):
            ro = g[f"e{e}_m{m}_row_off"]
            mm = g[f"e{e}_m{m}_minmax"]
            rows = len(ro) - 1
            cols = int(g["d_model"]) if m == 0 else int(g["d_ff"])
            c = q.CompressedMatrix(rows, cols, g[f"e{e}_m{m}_cw"], ro, mm, dic.hash64)
            lst.append(c)
    return wi, wo


def test_moe_tiny_matches_reference_golden(dic, golden):
    g = golden("moe_tiny.npz")
    wi, wo = layer_from_golden(g, dic)
    layer = q.CompressedMoELayer([c.to_device(dic) for c in wi], [c.to_device(dic) for c in wo], dic)
    assign = q.RouterSim(int(g["E"]), rule="argmax", seed=0).assign(g["x"])
    assert np.array_equal(assign, g["assign"])
    y = layer.forward(g["x"], assign)
    d = bf16_ulp_diff(y, g["y"])
    assert d.max() <= 2, d.max()
    assert np.mean(d == 0) >= 0.99


@pytest.mark.parametrize("T", [1, 3, 16, 64, 200])
def test_moe_random_layer_vs_oracle(dic, odic, T):
    rng = np.random.default_rng(T)
    E, d_model, d_ff = 8, 128, 512
    wi, wo, host = [], [], []
    for e in range(E):
        pair = []
        for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            t = q.rtn_quantize(w, q.make_grid(w))
            c = q.encode(t, dic)
            lst.append(c.to_device(dic))
            pair.append((rows, cols, c.codewords, c.row_off, c.row_minmax))
        host.append(tuple(pair))
    layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=4)
    layer.publish_plan = True  # the dispatcher outputs are checked below
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    assign = q.RouterSim(E, rule="argmax", seed=1, skew=0.5 if T > 50 else 0.0).assign(x)
    y = layer.forward(x, assign)
    y_ref = O.moe_layer(x, assign, host, odic)
    d = bf16_ulp_diff(y, y_ref)
    assert d.max() <= 2
    assert np.mean(d == 0) >= 0.99
    # expert grouping follows buffer order
    counts = layer.expert_count.cpu().numpy()
    assert np.array_equal(counts, np.bincount(assign, minlength=E))
    order = layer.order.cpu().numpy()[:T]
    want = np.concatenate([np.flatnonzero(assign == e) for e in range(E)])
    assert np.array_equal(order, want)


def test_host_forward_graph_replays_fresh_inputs(dic, odic):
    """forward() captures a per-T graph (H2D copy, step, y into pinned host
    memory) on first use; later calls replay it. Every call must see its own
    tokens and ids, and the returned array must not alias the next call's."""
    rng = np.random.default_rng(5)
    E, d_model, d_ff, T = 6, 128, 384, 24
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
    outs = []
    for call in range(4):
        x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
        assign = rng.integers(0, E, size=T).astype(np.int32)
        y = layer.forward(x, assign)
        outs.append((y, O.moe_layer(x, assign, host, odic)))
    assert any(st["graphs"].get(False) is not None for st in layer._stages.values())
    for y, y_ref in outs:  # earlier results intact after later calls
        d = bf16_ulp_diff(y, y_ref)
        assert d.max() <= 2
        assert np.mean(d == 0) >= 0.99


@pytest.mark.parametrize("T", [24, 96])
def test_forward_stream_equals_forward(dic, T):
    """The pipelined host API (two steps in flight, per-slot pinned buffers
    and graphs, layers alternating) returns, in order, exactly what one
    blocking forward() per step returns — no slot's inputs or outputs are
    overwritten while its step is in flight. T = 96 (16 tokens per expert)
    takes the decode-then-MMA path."""
    rng = np.random.default_rng(11)
    E, d_model, d_ff = 6, 128, 384
    layers = []
    for l in range(3):
        wi, wo = [], []
        for e in range(E):
            for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
                w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
                lst.append(q.encode(q.rtn_quantize(w, q.make_grid(w)), dic).to_device(dic))
        layers.append(q.CompressedMoELayer(wi, wo, dic, max_tokens=T))
    steps = []
    for i in range(11):
        x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
        steps.append((layers[i % 3], x, rng.integers(-1, E, size=T).astype(np.int32)))
    piped = list(q.forward_stream(iter(steps)))
    piped2 = list(q.forward_stream(iter(steps), depth=3))  # graphs captured: replays
    ref = [lay.forward(x, a) for lay, x, a in steps]
    assert len(piped) == len(steps)
    for y, y2, r in zip(piped, piped2, ref):
        assert np.array_equal(y, r) and np.array_equal(y2, r)


def test_moe_step_is_graph_capturable(dic):
    rng = np.random.default_rng(5)
    E, d_model, d_ff = 4, 64, 256
    mats = []
    for e in range(E):
        for rows, cols in ((d_ff, d_model), (d_model, d_ff)):
            w = torch.randn(rows, cols, device="cuda") * 0.02
            codes, mm = q.rtn_quantize_device(w)
            mats.append(q.encode_device(codes, mm, dic))
    layer = q.CompressedMoELayer(mats[0::2], mats[1::2], dic, max_tokens=32)
    x = torch.from_numpy(q.bf16_round(rng.normal(size=(32, d_model)).astype(np.float32))).cuda().to(torch.bfloat16)
    a = torch.from_numpy(rng.integers(0, E, 32).astype(np.int32)).cuda()
    out = torch.empty((32, d_model), device="cuda")
    ref = layer.forward_device(x, a).clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        layer.forward_device(x, a, out=out)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        layer.forward_device(x, a, out=out)
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_codebook_reindexing_is_exact(dic):
    """Frequency codebook: streams rewritten to ranks decode to the same codes
    and the packed table follows the permutation."""
    from paper_2310_16795_b200.codebook import Codebook
    from paper_2310_16795_b200.codec import decompress_device

    mats = []
    for k in range(3):
        w = torch.randn(300, 1024, device="cuda") * 0.02
        codes, mm = q.rtn_quantize_device(w)
        mats.append((codes, q.encode_device(codes, mm, dic)))
    cb = Codebook(dic, [m for _, m in mats])
    before = [m.cw.clone() for _, m in mats]
    cb.apply([m for _, m in mats])
    assert cb.hit_rate(40960) >= cb.counts[:40960].sum() / cb.counts.sum()
    for (codes, m), b in zip(mats, before):
        assert not torch.equal(m.cw, b)
        out, bad = decompress_device(m, dic)
        assert int(bad[0]) == 0
        assert torch.equal(out, codes)


@pytest.mark.parametrize("d_model,d_ff", [(256, 2048), (512, 8192)])
def test_moe_segmented_rows_vs_oracle(dic, odic, d_model, d_ff):
    """Long rows use G = 2^lg lanes per row with precomputed column
    checkpoints (lg = 1..3); outputs must still match the composed oracle."""
    rng = np.random.default_rng(d_ff)
    E = 3
    wi, wo, host = [], [], []
    for e in range(E):
        pair = []
        for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            t = q.rtn_quantize(w, q.make_grid(w))
            c = q.encode(t, dic)
            dm = q.DeviceMatrix.from_host(c, dic, torch.device("cuda", 0))
            lst.append(dm)
            pair.append((rows, cols, c.codewords, c.row_off, c.row_minmax))
        host.append(tuple(pair))
    layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=8)
    assert layer.lanes_per_row(7)[1] >= 1 or max(m.lg for m in wo) >= 1  # several lanes per wo row
    x = q.bf16_round(rng.normal(size=(7, d_model)).astype(np.float32))
    assign = np.array([0, 1, 2, 0, 0, 2, 1], np.int32)
    y = layer.forward(x, assign)
    y_ref = O.moe_layer(x, assign, host, odic)
    d = bf16_ulp_diff(y, y_ref)
    assert d.max() <= 2
    assert np.mean(d == 0) >= 0.99


@pytest.mark.parametrize("T", [40, 200])
def test_moe_dense_decode_then_mma_vs_oracle(dic, odic, T):
    """Batched regime: decode-then-MMA passes (qmoe_dense_moe_pass) — several
    row blocks, K chunks with straddling codewords, experts with 0, < 32 and
    > 64 tokens — against the composed oracle and the streaming path."""
    rng = np.random.default_rng(T + 7)
    E, d_model, d_ff = 4, 320, 1100  # 1100 rows: 3 row blocks (last partial); 320 cols: 5 chunks
    wi, wo, host = [], [], []
    for e in range(E):
        pair = []
        for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            t = q.rtn_quantize(w, q.make_grid(w))
            c = q.encode(t, dic)
            lst.append(c.to_device(dic))
            pair.append((rows, cols, c.codewords, c.row_off, c.row_minmax))
        host.append(tuple(pair))
    layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=T)
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    assign = np.where(np.arange(T) % 5 == 0, 1, rng.integers(0, 3, size=T)).astype(np.int32)  # expert 3: no tokens
    layer.dense_mode = "always"
    y = layer.forward(x, assign)
    y_ref = O.moe_layer(x, assign, host, odic)
    d = bf16_ulp_diff(y, y_ref)
    assert d.max() <= 2, d.max()
    assert np.mean(d == 0) >= 0.99
    layer.dense_mode = "never"
    y_stream = layer.forward(x, assign)
    assert bf16_ulp_diff(y, y_stream).max() <= 2


def _random_layer(dic, rng, E, d_model, d_ff, max_tokens):
    wi, wo, host = [], [], []
    for e in range(E):
        pair = []
        for rows, cols, lst in ((d_ff, d_model, wi), (d_model, d_ff, wo)):
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            t = q.rtn_quantize(w, q.make_grid(w))
            c = q.encode(t, dic)
            lst.append(c.to_device(dic))
            pair.append((rows, cols, c.codewords, c.row_off, c.row_minmax))
        host.append(tuple(pair))
    return wi, wo, host


@pytest.mark.parametrize("T", [1, 2, 5, 48, 100, 200, 300])
def test_fused_step_equals_grouped_passes_and_plan(dic, T):
    """The single-launch step (qmoe_moe_step) runs the same decode with the same
    lanes as the plan kernel + two grouped passes: outputs must be bit-identical,
    and its dispatcher outputs (stable per-expert order, counts) exact. T = 1, 2
    run the phase-split schedule (half the CTAs per phase)."""
    rng = np.random.default_rng(100 + T)
    E, d_model, d_ff = 6, 192, 640
    wi, wo, _ = _random_layer(dic, rng, E, d_model, d_ff, T)
    layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=T)
    layer.publish_plan = True
    assert layer.fused
    x = torch.from_numpy(q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))).cuda().to(torch.bfloat16)
    a_np = rng.integers(-1, E + 1, size=T).astype(np.int32)  # -1 and E: no expert (dropped)
    a = torch.from_numpy(a_np).cuda()
    y_fused = layer.forward_device(x, a).clone()
    ok = (a_np >= 0) & (a_np < E)
    order = np.argsort(np.where(ok, a_np, E), kind="stable")[: ok.sum()]
    assert np.array_equal(layer.order[: ok.sum()].cpu().numpy(), order)
    assert np.array_equal(layer.expert_count.cpu().numpy(), np.bincount(a_np[ok], minlength=E))
    layer2 = q.CompressedMoELayer(wi, wo, dic, max_tokens=T, fused=False)
    assert not layer2.fused
    y_grouped = layer2.forward_device(x, a)
    assert torch.equal(y_fused, y_grouped)  # incl. zero rows for tokens without an expert
    assert torch.all(y_fused[~torch.from_numpy(ok).cuda()] == 0)
    # later steps reuse the counters (two parity sets, no reset between steps):
    # alternate sizes and check every step against the first result
    half = max(1, T // 2)
    y_half_ref = layer2.forward_device(x[:half], a[:half]).clone()
    for it in range(5):
        if it % 2:
            assert torch.equal(layer.forward_device(x[:half], a[:half]), y_half_ref)
        else:
            assert torch.equal(layer.forward_device(x, a), y_fused)
    tickets = int(layer.counters[:2].cpu().numpy().view(np.int64)[0])
    assert tickets % 148 == 0 or tickets % torch.cuda.get_device_properties(0).multi_processor_count == 0


def test_fused_plan_many_experts(dic):
    """The fused step's warp plan sorts (expert, token) keys: with hundreds of
    experts (nothing in it scales with E) the stable order, counts and outputs
    still match the grouped path."""
    rng = np.random.default_rng(77)
    E, d_model, d_ff, T = 600, 64, 128, 160
    wi, wo, _ = _random_layer(dic, rng, E, d_model, d_ff, T)
    layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=T)
    layer.publish_plan = True
    assert layer.fused
    x = torch.from_numpy(q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))).cuda().to(torch.bfloat16)
    a_np = np.where(rng.random(T) < 0.5, rng.integers(0, 8, size=T), rng.integers(-2, E + 2, size=T)).astype(np.int32)
    a = torch.from_numpy(a_np).cuda()
    y_fused = layer.forward_device(x, a).clone()
    ok = (a_np >= 0) & (a_np < E)
    order = np.argsort(np.where(ok, a_np, E), kind="stable")[: ok.sum()]
    assert np.array_equal(layer.order[: ok.sum()].cpu().numpy(), order)
    assert np.array_equal(layer.expert_count.cpu().numpy(), np.bincount(a_np[ok], minlength=E))
    layer2 = q.CompressedMoELayer(wi, wo, dic, max_tokens=T, fused=False)
    y_grouped = layer2.forward_device(x, a)
    assert torch.equal(y_fused[ok], y_grouped[ok])


def test_empty_step_and_no_expert_tokens(dic):
    """T = 0 through the host API and the device API; a step whose tokens all
    lack an expert (ids outside [0, E)) returns zero rows on the host API."""
    rng = np.random.default_rng(3)
    E, d_model, d_ff = 4, 64, 128
    wi, wo, _ = _random_layer(dic, rng, E, d_model, d_ff, 8)
    layer = q.CompressedMoELayer(wi, wo, dic, max_tokens=8)
    y0 = layer.forward(np.zeros((0, d_model), np.float32), np.zeros(0, np.int32))
    assert y0.shape == (0, d_model)
    yd = layer.forward_device(torch.zeros((0, d_model), device="cuda"), torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert tuple(yd.shape) == (0, d_model)
    x = q.bf16_round(rng.normal(size=(5, d_model)).astype(np.float32))
    ids = np.array([-1, E, E + 7, -3, -1], np.int32)
    y = layer.forward(x, ids)
    assert y.shape == (5, d_model) and np.all(y == 0)  # no expert: zero rows, as the composed reference
    mixed = np.array([0, -1, 2, E, 1], np.int32)
    ym = layer.forward(x, mixed)
    assert np.all(ym[[1, 3]] == 0) and np.any(ym[[0, 2, 4]] != 0)


def test_dense_pass_ignores_row_padding(dic, odic):
    """The hidden rows are padded to a 16-byte stride and the padding is never
    written: the decode-then-MMA pass must not read it into the MMA (NaN bit
    patterns there would poison whole accumulators: 0 * NaN = NaN)."""
    rng = np.random.default_rng(41)
    E, d_model, d_ff, T = 3, 96, 300, 90  # d_ff % 8 != 0: padded hidden rows
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
    assert layer.h.stride(0) > d_ff
    layer.h.fill_(float("nan"))
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    assign = rng.integers(0, E, size=T).astype(np.int32)
    layer.dense_mode = "always"
    y = layer.forward_device(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(assign).cuda())
    y_ref = O.moe_layer(x, assign, host, odic)
    d = bf16_ulp_diff(y.cpu().numpy(), y_ref)
    assert np.isfinite(y.cpu().numpy()).all()
    assert d.max() <= 2 and np.mean(d == 0) >= 0.99
