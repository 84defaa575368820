"""Per-kernel parity of libtcb200 (b200 dialect, cuda:0) against the CPU oracle.

Bar (BASELINE.json north_star): integer / index / layout work and
every reference op whose ref kernel has a fixed f32 order is BIT-EXACT; floating
point with a different association order (tensor-core GEMMs, parallel row
reductions) is checked with the tolerance written in each test.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gpu_util import bits_equal, max_ulp_bf16, quantize, rel_err, run_both  # noqa: E402

# bf16 outputs: both sides round (nearly) the same f32 values; near-zero
# cancellation makes ulp distance meaningless, so bf16 outputs are compared
# norm-wise against the bf16 epsilon (2^-8).
BF16_TOL = 4e-3
from paper_2303_04759_b200.abi import BF16, F16, F32, I32  # noqa: E402

RNG = np.random.default_rng(1234)


def rn(*shape, lo=-1.0, hi=1.0):
    return RNG.uniform(lo, hi, size=shape).astype(np.float32)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2303_04759_b200.runtime import lib
    lib()  # fail loudly if the extension is missing


# ---------------------------------------------------------------- elementwise

@pytest.mark.parametrize("dt", [F32, F16, BF16])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "tanh_dx"])
def test_binary_bit_exact(op, dt):
    a, b = rn(37, 53), rn(37, 53, lo=0.5, hi=2.0)
    for bshape in [(37, 53), (53,), (1,), (37, 1)]:
        bb = rn(*bshape, lo=0.5, hi=2.0)
        g, o = run_both(op, [(a, dt), (bb, dt)], [((37, 53), dt)])
        assert bits_equal(g[0], o[0]), (op, dt, bshape)
    g, o = run_both(op, [(rn(4, 1, 6), dt), (rn(3, 1, lo=0.5), dt)], [((4, 3, 6), dt)])
    assert bits_equal(g[0], o[0])


@pytest.mark.parametrize("dt", [F32, BF16])
@pytest.mark.parametrize("op", ["neg", "relu", "gtz"])
def test_unary_bit_exact(op, dt):
    g, o = run_both(op, [(rn(1000, lo=-3, hi=3), dt)], [((1000,), dt)])
    assert bits_equal(g[0], o[0])


@pytest.mark.parametrize("op", ["tanh", "gelu"])
def test_transcendental_unary(op):
    # device tanhf/erff vs glibc: a few f32 ulps
    g, o = run_both(op, [(rn(4096, lo=-4, hi=4), F32)], [((4096,), F32)])
    assert np.max(np.abs(g[0] - o[0])) <= 4e-7 * np.maximum(1, np.abs(o[0])).max()
    g, o = run_both(op, [(rn(4096, lo=-4, hi=4), BF16)], [((4096,), BF16)])
    assert max_ulp_bf16(g[0], o[0]) <= 1


def test_gelu_dx():
    g, o = run_both("gelu_dx", [(rn(2048, lo=-4, hi=4), F32), (rn(2048), F32)], [((2048,), F32)])
    assert rel_err(g[0], o[0]) < 1e-6


def test_layout_ops_bit_exact():
    x = rn(33, 65, lo=-100, hi=100)
    for to, dt in [("f16", F16), ("bf16", BF16), ("f32", F32)]:
        op = "cast" if to != "bf16" else "convert"
        g, o = run_both(op, [(x, F32)], [((33, 65), dt)], {"to": to})
        assert bits_equal(g[0], o[0])
    g, o = run_both("bcast", [(rn(65), F32)], [((3, 33, 65), F32)], {"shape": "3,33,65"})
    assert bits_equal(g[0], o[0])
    for dt in (F32, BF16):
        g, o = run_both("transpose", [(x, dt)], [((65, 33), dt)])
        assert bits_equal(g[0], o[0])
    g, o = run_both("reshape", [(x, F32)], [((65, 33), F32)], {"shape": "65,33"})
    assert bits_equal(g[0], o[0])
    g, o = run_both("view", [(x, F32)], [((7, 10), F32)], {"offset": 100, "shape": "7,10"})
    assert bits_equal(g[0], o[0])


def test_dropout_mask_bit_exact():
    x = rn(10007)
    for p in (0.0, 0.1, 0.5):
        attrs = {"p": p, "seed": 7, "salt": 3}
        g, o = run_both("dropout", [(x, F32)], [((10007,), F32)], attrs)
        assert bits_equal(g[0], o[0]), p
        g, o = run_both("dropout", [(x, BF16)], [((10007,), BF16)], attrs)
        assert bits_equal(g[0], o[0]), p


# ------------------------------------------------------------------ reductions

@pytest.mark.parametrize("op", ["sum", "mean"])
def test_reductions_exact(op):
    x = rn(6, 50, 7)
    for axes, shape in [("", (1,)), ("0", (50, 7)), ("1", (6, 7)), ("2", (6, 50)), ("0,2", (50,))]:
        g, o = run_both(op, [(x, F32)], [(shape, F32)], {"axes": axes})
        assert bits_equal(g[0], o[0]), axes
    g, o = run_both(op, [(rn(300, 96), F16)], [((96,), F16)], {"axes": "0"})
    assert bits_equal(g[0], o[0])


def test_reduction_bf16_fast_path():
    x = rn(4096, 768)
    g, o = run_both("sum", [(x, BF16)], [((768,), F32)], {"axes": "0"})
    assert rel_err(g[0], o[0]) < 1e-5
    g, o = run_both("mean", [(x, BF16)], [((4096,), F32)], {"axes": "1"})
    assert rel_err(g[0], o[0]) < 1e-5


@pytest.mark.parametrize("shape", [(4096, 768), (300, 2304), (77, 40)])
def test_colsum(shape):
    x = rn(*shape)
    g, o = run_both("colsum", [(x, BF16)], [((shape[1],), F32)])
    assert rel_err(g[0], o[0]) < 1e-5
    g, o = run_both("colsum", [(x, F32)], [((shape[1],), F32)])
    assert bits_equal(g[0], o[0])  # f32: exact row order


@pytest.mark.parametrize("shape", [(4096, 30528), (300, 2304), (77, 40)])
def test_colsum_masked(shape):
    """colsum(x, labels) skips rows labelled ignore_index (the CE gradient's
    exact-zero rows); the oracle adds the masked-out rows' zeros instead."""
    R, C = shape
    x = rn(R, C)
    lab = RNG.integers(0, 50, size=R).astype(np.int32)
    lab[RNG.uniform(size=R) < 0.85] = -100
    x[lab == -100] = 0.0  # what the CE gradient holds there
    g, o = run_both("colsum", [(x, BF16), (lab, I32)], [((C,), F32)], {"ignore_index": -100})
    assert rel_err(g[0], o[0]) < 1e-5


def test_embedding_dx_single_long_segment():
    """token-type ids: every token hits row 0 (one 4096-long segment).  Long
    segments are folded in 128-row chunks (deterministic, not the oracle's
    single sequential chain): norm-wise 1e-6; segments <= 128 stay bit-exact."""
    T, H = 4096, 768
    ids = np.zeros(T, np.int32)
    dy = rn(T, H)
    g, o = run_both("embedding_dx", [(ids, I32), (dy, BF16)], [((2, H), F32)], {"rows": 2})
    assert rel_err(g[0], o[0]) < 1e-6
    ids = (np.arange(T) % 32).astype(np.int32)  # 32 segments of exactly 128
    g, o = run_both("embedding_dx", [(ids, I32), (dy, BF16)], [((32, H), F32)], {"rows": 32})
    assert bits_equal(g[0], o[0])


@pytest.mark.parametrize("T,V,kind", [(5000, 30000, "random"), (4100, 2, "zeros"), (3000, 70000, "random"),
                                      (70000, 512, "positions"), (257, 1, "zeros")])
def test_embedding_dx_radix_sorted_segments(T, V, kind):
    """The stable LSD radix sort behind embedding_dx (1, 2 and 3 digit passes,
    ragged tiles): segments of <= 128 equal ids are the oracle's sequential
    sums bit for bit, longer ones within 1e-6 (chunked fold)."""
    H = 96
    rng = np.random.default_rng(T + V)
    if kind == "random":
        ids = rng.integers(0, V, T).astype(np.int32)
    elif kind == "zeros":
        ids = np.zeros(T, np.int32)
    else:
        ids = (np.arange(T) % V).astype(np.int32)
    dy = rn(T, H)
    g, o = run_both("embedding_dx", [(ids, I32), (dy, F32)], [((V, H), F32)], {"rows": V})
    longest = np.bincount(ids, minlength=V).max()
    if longest <= 128:
        assert bits_equal(g[0], o[0])
    else:  # a different f32 summation order over `longest` terms: ~sqrt(n) eps relative
        exact = np.zeros((V, H))
        np.add.at(exact, ids, dy.astype(np.float64))
        assert rel_err(g[0], exact) < 1e-5 and rel_err(o[0], exact) < 1e-5


def test_mse_exact():
    g, o = run_both("mse", [(rn(64, 10), F32), (rn(64, 10), F32)], [((1,), F32)])
    assert bits_equal(g[0], o[0])


# ------------------------------------------------------------------------ gemm

@pytest.mark.parametrize("mnk", [(2, 4, 3), (33, 47, 65), (128, 96, 64)])
@pytest.mark.parametrize("dt", [F32, F16])
def test_matmul_exact_kernel_bit_exact(mnk, dt):
    m, n, k = mnk
    g, o = run_both("matmul", [(rn(m, k), dt), (rn(k, n), dt)], [((m, n), dt)])
    assert bits_equal(g[0], o[0])


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("mnk", [(128, 128, 64), (300, 200, 136), (256, 512, 1024), (1000, 768, 320)])
def test_matmul_t_tcgen05(mnk, ta, tb):
    """bf16 tcgen05 GEMM, f32 output: only the fp32 summation order differs from
    the oracle's k-ascending loop -> norm-wise rel err < 1e-5."""
    m, n, k = mnk
    a = rn(k, m) if ta else rn(m, k)
    b = rn(n, k) if tb else rn(k, n)
    attrs = {"ta": ta, "tb": tb, "alpha": 0.5}
    g, o = run_both("matmul_t", [(a, BF16), (b, BF16)], [((m, n), F32)], attrs)
    assert rel_err(g[0], o[0]) < 1e-5, rel_err(g[0], o[0])
    g, o = run_both("matmul_t", [(a, BF16), (b, BF16)], [((m, n), BF16)], attrs)
    assert rel_err(g[0], o[0]) < BF16_TOL


TILES = [(256, 2), (192, 2), (128, 2), (256, 1), (192, 1), (128, 1)]


@pytest.mark.parametrize("bn,cg", TILES)
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("mnk", [(256, 256, 128), (520, 328, 200), (1000, 768, 320)])
def test_gemm_tile_variants(mnk, ta, tb, bn, cg):
    """Every tcgen05 tile configuration (1-CTA and CTA-pair, all operand
    majors, ragged M/N/K tails) against the oracle, f32 and bf16 outputs."""
    m, n, k = mnk
    a = rn(k, m) if ta else rn(m, k)
    b = rn(n, k) if tb else rn(k, n)
    attrs = {"ta": ta, "tb": tb, "alpha": 0.5, "tc_bn": bn, "tc_cg": cg}
    g, o = run_both("matmul_t", [(a, BF16), (b, BF16)], [((m, n), F32)], attrs)
    assert rel_err(g[0], o[0]) < 1e-5, rel_err(g[0], o[0])
    g, o = run_both("matmul_t", [(a, BF16), (b, BF16)], [((m, n), BF16)], attrs)
    assert rel_err(g[0], o[0]) < BF16_TOL


@pytest.mark.parametrize("bn,cg", TILES)
def test_gemm_tile_variants_epilogues(bn, cg):
    """bias + GeLU + saved pre-activation, and the fused act'(aux) dgrad
    epilogue (aux arrives by TMA), for every tile configuration."""
    m, k, n = 700, 256, 600
    x, w, bias = rn(m, k), rn(k, n, lo=-0.1, hi=0.1), rn(n)
    at = {"act": "gelu", "tc_bn": bn, "tc_cg": cg}
    g, o = run_both("linear", [(x, BF16), (w, BF16), (bias, F32)], [((m, n), BF16), ((m, n), BF16)], at)
    assert rel_err(g[0], o[0]) < BF16_TOL and rel_err(g[1], o[1]) < BF16_TOL
    g, o = run_both("linear", [(x, BF16), (w, BF16), (bias, BF16)], [((m, n), BF16)], at)
    assert rel_err(g[0], o[0]) < BF16_TOL
    dy, w2, u = rn(m, k), rn(n, k), rn(m, n, lo=-3, hi=3)
    g, o = run_both("matmul_dact", [(dy, BF16), (w2, BF16), (u, BF16)], [((m, n), BF16)],
                    {"tb": 1, "act": "gelu", "tc_bn": bn, "tc_cg": cg})
    assert rel_err(g[0], o[0]) < BF16_TOL


EPI_VARIANTS = [
    # (op, inputs (shape, dtype), outputs, attrs): the compile-time epilogue variants of k_gemm_tc
    ("matmul_t", [((700, 256), BF16), ((256, 600), BF16)], [((700, 600), BF16)], {}),  # plain bf16
    ("matmul_t", [((256, 700), BF16), ((256, 600), BF16)], [((700, 600), F32)], {"ta": 1, "out": "f32"}),  # f32
    ("linear", [((700, 256), BF16), ((256, 600), BF16), ((600,), F32)], [((700, 600), BF16)], {}),  # + bias
    ("linear", [((700, 256), BF16), ((256, 600), BF16), ((600,), F32)], [((700, 600), BF16)] * 2,
     {"act": "gelu", "save_preact": 1, "save": "grad"}),  # + bias + GELU + GELU' saved
    ("matmul_dact", [((700, 256), BF16), ((600, 256), BF16), ((700, 600), BF16)], [((700, 600), BF16)],
     {"tb": 1, "act": "deriv"}),  # * act'(aux)
    ("matmul_pair", [((512, 768), BF16), ((3072, 768), BF16), ((512, 3072), BF16), ((512, 3072), BF16),
                     ((512, 768), BF16)], [((512, 3072), BF16), ((3072, 768), F32)],
     {"n0": 3, "act0": "deriv", "ta0": 0, "tb0": 1, "ta1": 1, "tb1": 0, "out1": "f32", "wsplit": 2}),
]


@pytest.mark.parametrize("case", range(len(EPI_VARIANTS)))
def test_gemm_epilogue_variants_bit_identical_to_generic(case):
    """Each compile-time epilogue variant (plain, f32, bias, bias+GELU+GELU',
    act'(aux), and a grouped pair with K-slice partials) gives exactly the
    bits of the runtime-dispatched epilogue it replaces (tc_generic_epi=1),
    on ragged shapes; both against the oracle within bf16 rounding."""
    from gpu_util import from_torch, to_torch
    from paper_2303_04759_b200.runtime import run_op
    op, ins, outs, at = EPI_VARIANTS[case]
    xs = [rn(*shp, lo=-1, hi=1) for shp, _ in ins]
    tin = [to_torch(quantize(x, d), d) for x, (_, d) in zip(xs, ins)]
    fast = [from_torch(t) for t in run_op(op, tin, outs, at)]
    slow = [from_torch(t) for t in run_op(op, tin, outs, {**at, "tc_generic_epi": 1})]
    for a, b in zip(fast, slow):
        assert bits_equal(a, b)
    _, o = run_both(op, [(x, d) for x, (_, d) in zip(xs, ins)], outs, at)
    for a, b in zip(fast, o):
        assert rel_err(a, b) < 1e-2, rel_err(a, b)


def test_matmul_t_exact_flag_bit_exact():
    a, b = rn(70, 40), rn(40, 50)
    g, o = run_both("matmul_t", [(a, BF16), (b, BF16)], [((70, 50), BF16)], {"exact": 1})
    assert bits_equal(g[0], o[0])


@pytest.mark.parametrize("act", ["none", "relu", "tanh", "gelu"])
def test_linear_tcgen05(act):
    m, k, n = 512, 256, 384
    x, w, b = rn(m, k), rn(k, n, lo=-0.1, hi=0.1), rn(n)
    g, o = run_both("linear", [(x, BF16), (w, BF16), (b, F32)], [((m, n), BF16), ((m, n), BF16)],
                    {"act": act})
    assert rel_err(g[0], o[0]) < BF16_TOL and rel_err(g[1], o[1]) < BF16_TOL


@pytest.mark.parametrize("act", ["none", "relu", "tanh"])
def test_linear_f32_matches_matmul_add_act(act):
    """fp32 linear = opt-dialect matmul_add_act (bit-exact for none/relu)."""
    m, k, n = 64, 48, 80
    g, o = run_both("linear", [(rn(m, k), F32), (rn(k, n), F32), (rn(n), F32)], [((m, n), F32)],
                    {"act": act})
    if act == "tanh":
        assert rel_err(g[0], o[0]) < 1e-6
    else:
        assert bits_equal(g[0], o[0])


def test_matmul_dact_gelu():
    m, k, n = 256, 384, 192
    dy, w, u = rn(m, k), rn(n, k), rn(m, n, lo=-3, hi=3)
    g, o = run_both("matmul_dact", [(dy, BF16), (w, BF16), (u, BF16)], [((m, n), BF16)],
                    {"tb": 1, "act": "gelu"})
    assert rel_err(g[0], o[0]) < BF16_TOL


def test_batch_matmul():
    a, b = rn(6, 128, 64), rn(6, 128, 64)
    g, o = run_both("batch_matmul", [(a, BF16), (b, BF16)], [((6, 128, 128), F32)], {"tb": 1})
    assert rel_err(g[0], o[0]) < 1e-5
    g, o = run_both("batch_matmul", [(a, F32), (b, F32)], [((6, 128, 128), F32)], {"tb": 1})
    assert bits_equal(g[0], o[0])


# ------------------------------------------------------------------ optimizer

def test_sgd_bit_exact():
    g, o = run_both("sgd_update", [(rn(10001), F32), (rn(10001), F32)], [((10001,), F32)], {"lr": 0.01})
    assert bits_equal(g[0], o[0])


def test_adam_double_math():
    n = 100003
    p, gr, m, v = rn(n), rn(n), rn(n, lo=-0.1, hi=0.1), rn(n, lo=0, hi=0.01)
    attrs = {"lr": 1e-3, "beta1": 0.9, "beta2": 0.999, "eps": 1e-6}
    step = np.array([3.0], np.float32)
    g, o = run_both("adam_update", [(p, F32), (gr, F32), (m, F32), (v, F32), (step, F32)],
                    [((n,), F32)] * 3, attrs)
    for x, y in zip(g, o):
        # double math on both sides; only the device pow() ulp in 1-beta^t differs
        assert np.max(np.abs(x - y) / np.maximum(np.abs(y), 1e-30)) < 2e-7
    g, o = run_both("adam_update_ex", [(p, F32), (gr, F32), (m, F32), (v, F32), (step, F32)],
                    [((n,), F32)] * 3 + [((n,), BF16)], dict(attrs, grad_scale=0.25))
    assert rel_err(g[3], o[3]) < BF16_TOL and rel_err(g[0], o[0]) < 1e-7


# ------------------------------------------------------------ transformer ops

@pytest.mark.parametrize("dt,H", [(F32, 128), (BF16, 768), (BF16, 1000)])
def test_layer_norm(dt, H):
    T = 257
    x, gm, bt = rn(T, H, lo=-2, hi=2), rn(H, lo=0.5, hi=1.5), rn(H, lo=-0.1, hi=0.1)
    g, o = run_both("layer_norm", [(x, dt), (gm, F32), (bt, F32)], [((T, H), dt), ((T,), F32), ((T,), F32)],
                    {"eps": 1e-12})
    assert rel_err(g[1], o[1]) < 1e-5 and rel_err(g[2], o[2]) < 1e-5
    if dt == F32:
        assert rel_err(g[0], o[0]) < 1e-5
    else:
        assert rel_err(g[0], o[0]) < BF16_TOL


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_add_layer_norm_and_backward(p):
    T, H = 300, 768
    x, r = rn(T, H), rn(T, H)
    gm, bt = rn(H, lo=0.5, hi=1.5), rn(H, lo=-0.1, hi=0.1)
    attrs = {"eps": 1e-12, "p": p, "seed": 11, "salt": 5}
    g, o = run_both("add_layer_norm", [(x, BF16), (r, BF16), (gm, F32), (bt, F32)],
                    [((T, H), BF16), ((T, H), BF16), ((T,), F32), ((T,), F32)], attrs)
    assert bits_equal(g[1], o[1])  # s = round(dropout(x) + r): bit-exact incl. the Philox mask
    assert rel_err(g[0], o[0]) < BF16_TOL
    s, mean, rstd = o[1], o[2], o[3]
    dy, dy2 = rn(T, H), rn(T, H)
    g, o = run_both("layer_norm_dx", [(s, BF16), (gm, F32), (mean, F32), (rstd, F32), (dy, BF16), (dy2, BF16)],
                    [((T, H), BF16), ((H,), F32), ((H,), F32), ((T, H), BF16)], attrs)
    assert rel_err(g[0], o[0]) < 5e-3 and rel_err(g[3], o[3]) < 5e-3
    assert rel_err(g[1], o[1]) < 1e-5 and rel_err(g[2], o[2]) < 1e-5
    # fused bias gradient (graph pattern 4): column sums of the outgoing gradient
    outs = [((T, H), BF16), ((H,), F32), ((H,), F32), ((T, H), BF16), ((H,), F32)]
    g, o = run_both("layer_norm_dx", [(s, BF16), (gm, F32), (mean, F32), (rstd, F32), (dy, BF16), (dy2, BF16)],
                    outs, {**attrs, "bias_grad": 1})
    # the column sums inherit the bf16 rounding differences of dx (5e-3 norm-wise)
    assert rel_err(g[4], o[4]) < 1e-4, rel_err(g[4], o[4])
    assert rel_err(g[3], o[3]) < 5e-3 and rel_err(g[1], o[1]) < 1e-5
    g, o = run_both("layer_norm_dx", [(s, BF16), (gm, F32), (mean, F32), (rstd, F32), (dy, BF16)],
                    outs[:3] + outs[4:], {**attrs, "p": 0.0, "bias_grad": 1})
    assert rel_err(g[3], o[3]) < 1e-4 and rel_err(g[0], o[0]) < 5e-3


@pytest.mark.parametrize("H,gdt", [(768, BF16), (1000, F32), (1000, BF16), (256, F32), (2048, F32)])
def test_layer_norm_fwd_bwd_shapes(H, gdt):
    # ragged row count (tail CTA with dead warps / a half-filled warp), 16-bit
    # and f32 gamma/beta, full and partial last chunks, the largest supported H
    T = 77
    x, r = rn(T, H), rn(T, H)
    gm, bt = rn(H, lo=0.5, hi=1.5), rn(H, lo=-0.1, hi=0.1)
    attrs = {"eps": 1e-12, "p": 0.1, "seed": 3, "salt": 9}
    g, o = run_both("add_layer_norm", [(x, BF16), (r, BF16), (gm, gdt), (bt, gdt)],
                    [((T, H), BF16), ((T, H), BF16), ((T,), F32), ((T,), F32)], attrs)
    assert bits_equal(g[1], o[1])
    assert rel_err(g[0], o[0]) < BF16_TOL and rel_err(g[2], o[2]) < 1e-5 and rel_err(g[3], o[3]) < 1e-5
    s, mean, rstd = o[1], o[2], o[3]
    dy, dy2 = rn(T, H), rn(T, H)
    outs = [((T, H), BF16), ((H,), F32), ((H,), F32), ((T, H), BF16), ((H,), F32)]
    g, o = run_both("layer_norm_dx", [(s, BF16), (gm, gdt), (mean, F32), (rstd, F32), (dy, BF16), (dy2, BF16)],
                    outs, {**attrs, "bias_grad": 1})
    assert rel_err(g[0], o[0]) < 5e-3 and rel_err(g[3], o[3]) < 5e-3
    assert rel_err(g[1], o[1]) < 1e-5 and rel_err(g[2], o[2]) < 1e-5 and rel_err(g[4], o[4]) < 1e-4


@pytest.mark.parametrize("T", [77, 300])
def test_layer_norm_saved_dropout_mask(T):
    """add_layer_norm(save_mask) writes the residual-branch keep bits (one byte
    per 8 elements, bit-exact vs the oracle's Philox draws); layer_norm_dx
    (mask_in) reading them gives bit-identical gradients to re-running Philox."""
    H = 768
    x, r = rn(T, H), rn(T, H)
    gm, bt = rn(H, lo=0.5, hi=1.5), rn(H, lo=-0.1, hi=0.1)
    attrs = {"eps": 1e-12, "p": 0.1, "seed": 5, "salt": 17}
    n32 = T * H // 32
    g, o = run_both("add_layer_norm", [(x, BF16), (r, BF16), (gm, BF16), (bt, BF16)],
                    [((T, H), BF16), ((T, H), BF16), ((T,), F32), ((T,), F32), ((n32,), I32)],
                    {**attrs, "save_mask": 1})
    assert bits_equal(g[1], o[1]) and np.array_equal(g[4].view(np.uint8), o[4].view(np.uint8))
    keep = np.unpackbits(g[4].view(np.uint8), bitorder="little")[: T * H]
    from oracle import oracle_py as O
    assert np.array_equal(keep, O.dropout_keep_mask(5, 17, T * H, 0.1))
    s, mean, rstd, mask = o[1], o[2], o[3], g[4]
    dy, dy2 = rn(T, H), rn(T, H)
    outs = [((T, H), BF16), ((H,), F32), ((H,), F32), ((T, H), BF16)]
    ins = [(s, BF16), (gm, BF16), (mean, F32), (rstd, F32), (dy, BF16), (dy2, BF16)]
    g1, o1 = run_both("layer_norm_dx", ins + [(mask, I32)], outs, {**attrs, "mask_in": 1})
    g0, _ = run_both("layer_norm_dx", ins, outs, attrs)
    for a, b in zip(g1, g0):
        assert bits_equal(a, b)
    assert rel_err(g1[3], o1[3]) < 5e-3 and rel_err(g1[1], o1[1]) < 1e-5


def test_layer_norm_dx_f32():
    T, H = 64, 128
    s, gm = rn(T, H), rn(H, lo=0.5, hi=1.5)
    mean = s.mean(1).astype(np.float32)
    rstd = (1 / np.sqrt(s.var(1) + 1e-12)).astype(np.float32)
    g, o = run_both("layer_norm_dx", [(s, F32), (gm, F32), (mean, F32), (rstd, F32), (rn(T, H), F32)],
                    [((T, H), F32), ((H,), F32), ((H,), F32)])
    for a, b in zip(g, o):
        assert rel_err(a, b) < 1e-5


@pytest.mark.parametrize("causal", [0, 1])
def test_softmax_and_dx(causal):
    x = rn(4, 128, 128, lo=-5, hi=5)
    g, o = run_both("softmax", [(x, F32)], [((4, 128, 128), F32)], {"scale": 0.125, "causal": causal})
    assert rel_err(g[0], o[0]) < 1e-6
    y, dy = o[0], rn(4, 128, 128)
    g, o = run_both("softmax_dx", [(y, F32), (dy, F32)], [((4, 128, 128), F32)], {"scale": 0.125})
    assert rel_err(g[0], o[0]) < 1e-5


@pytest.mark.parametrize("dt", [F32, BF16])
@pytest.mark.parametrize("p,causal", [(0.0, 0), (0.1, 0), (0.0, 1)])
def test_attention_fwd_bwd(dt, p, causal):
    B, S, A, dh = 2, 128, 4, 64
    H = A * dh
    T = B * S
    qkv = rn(T, 3 * H)
    attrs = {"heads": A, "seq": S, "p": p, "seed": 3, "salt": 9, "causal": causal}
    g, o = run_both("attention", [(qkv, dt)], [((T, H), dt), ((B * A * S, S), dt)], attrs)
    tol = 1e-5 if dt == F32 else 2e-2
    assert rel_err(g[0], o[0]) < tol and rel_err(g[1], o[1]) < tol, (rel_err(g[0], o[0]), rel_err(g[1], o[1]))
    probs, dctx = o[1], rn(T, H)
    g, o = run_both("attention_dx", [(qkv, dt), (probs, dt), (dctx, dt)], [((T, 3 * H), dt)], attrs)
    assert rel_err(g[0], o[0]) < (1e-5 if dt == F32 else 3e-2), rel_err(g[0], o[0])


@pytest.mark.parametrize("S", [128, 72, 40])
@pytest.mark.parametrize("p,causal", [(0.0, 0), (0.1, 0), (0.1, 1)])
def test_attention_fused_tcgen05(S, p, causal):
    """Fused tcgen05 attention (one CTA per head, S <= 128, dh 64) against the
    oracle and against the unfused GEMM + row-softmax path on the GPU."""
    B, A, dh = 3, 2, 64
    H, T = A * dh, B * S
    qkv = rn(T, 3 * H, lo=-2, hi=2)
    at = {"heads": A, "seq": S, "p": p, "seed": 5, "salt": 11, "causal": causal}
    outs = [((T, H), BF16), ((B * A * S, S), BF16)]
    g, o = run_both("attention", [(qkv, BF16)], outs, at)
    assert rel_err(g[1], o[1]) < 1e-2, rel_err(g[1], o[1])
    assert rel_err(g[0], o[0]) < 2e-2, rel_err(g[0], o[0])
    gu, _ = run_both("attention", [(qkv, BF16)], outs, {**at, "unfused": 1})
    assert rel_err(g[0], gu[0]) < 1e-2 and rel_err(g[1], gu[1]) < 1e-2
    probs, dctx = o[1], rn(T, H)
    ins = [(qkv, BF16), (probs, BF16), (dctx, BF16)]
    g, o = run_both("attention_dx", ins, [((T, 3 * H), BF16)], at)
    assert rel_err(g[0], o[0]) < 3e-2, rel_err(g[0], o[0])
    gu, _ = run_both("attention_dx", ins, [((T, 3 * H), BF16)], {**at, "unfused": 1})
    assert rel_err(g[0], gu[0]) < 2e-2, rel_err(g[0], gu[0])


@pytest.mark.parametrize("S,causal", [(128, 0), (64, 1)])
def test_attention_saved_dropout_mask(S, causal):
    """attention(save_mask) writes the keep bits of its P dropout (4 words per
    query row, bit-exact vs the oracle); attention_dx reading them equals the
    Philox re-run bit for bit."""
    B, A, dh = 2, 2, 64
    H, T = A * dh, B * S
    qkv = rn(T, 3 * H, lo=-2, hi=2)
    at = {"heads": A, "seq": S, "p": 0.1, "seed": 9, "salt": 4, "causal": causal}
    outs = [((T, H), BF16), ((B * A * S, S), BF16)]
    nw = B * A * S * 4
    g, o = run_both("attention", [(qkv, BF16)], outs + [((nw,), I32)], {**at, "save_mask": 1})
    g0, _ = run_both("attention", [(qkv, BF16)], outs, at)
    assert bits_equal(g[0], g0[0]) and bits_equal(g[1], g0[1])
    # words hold bits for keys 0..127; only keys < S are meaningful
    gw, ow = g[2].view(np.uint32).reshape(-1, 4), o[2].view(np.uint32).reshape(-1, 4)
    keymask = np.array([(1 << 32) - 1 if (w + 1) * 32 <= S else ((1 << max(0, S - 32 * w)) - 1)
                        for w in range(4)], dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(gw & keymask, ow & keymask)
    probs, dctx = o[1], rn(T, H)
    ins = [(qkv, BF16), (probs, BF16), (dctx, BF16)]
    g1, o1 = run_both("attention_dx", ins + [(g[2], I32)], [((T, 3 * H), BF16)], at)
    g2, _ = run_both("attention_dx", ins, [((T, 3 * H), BF16)], at)
    assert bits_equal(g1[0], g2[0])
    assert rel_err(g1[0], o1[0]) < 3e-2


def test_embedding_bit_exact():
    V, H, T = 1000, 96, 513
    ids = RNG.integers(0, V, size=T).astype(np.int32)
    ids[:40] = 7  # collisions
    table = rn(V, H)
    for dt in (F32, BF16):
        g, o = run_both("embedding", [(ids, I32), (table, dt)], [((T, H), dt)])
        assert bits_equal(g[0], o[0])
    dy = rn(T, H)
    g, o = run_both("embedding_dx", [(ids, I32), (dy, F32)], [((V, H), F32)])
    assert bits_equal(g[0], o[0])  # deterministic ordered scatter-add == oracle order
    base = rn(V, H)
    g, o = run_both("embedding_dx", [(ids, I32), (dy, BF16), (base, F32)], [((V, H), F32)])
    assert bits_equal(g[0], o[0])


@pytest.mark.parametrize("dt", [F32, BF16])
def test_cross_entropy(dt):
    T, V, Vp = 300, 1000, 1024
    x = rn(T, Vp, lo=-4, hi=4)
    lab = RNG.integers(0, V, size=T).astype(np.int32)
    lab[::7] = -100
    attrs = {"classes": V, "ignore_index": -100}
    g, o = run_both("cross_entropy", [(x, dt), (lab, I32)], [((1,), F32), ((T, Vp), dt)], attrs)
    assert abs(g[0][0] - o[0][0]) <= 1e-5 * abs(o[0][0])
    assert rel_err(g[1], o[1]) < (1e-5 if dt == F32 else 5e-3)
    assert np.all(g[1][:, V:] == 0) and np.all(g[1][::7] == 0)


@pytest.mark.parametrize("dt", [F32, BF16])
def test_cross_entropy_in_place(dt):
    """The planner runs cross_entropy in place (dlogits overwrite the logits):
    bit-identical to separate buffers, label logits included."""
    import torch
    from gpu_util import from_torch, to_torch
    from paper_2303_04759_b200.runtime import run_op
    T, V, Vp = 300, 1000, 1024
    x = rn(T, Vp, lo=-4, hi=4)
    lab = RNG.integers(0, V, size=T).astype(np.int32)
    lab[::5] = -100
    attrs = {"classes": V, "ignore_index": -100}
    xs, ls = to_torch(x, dt), to_torch(lab, I32)
    sep = [from_torch(t) for t in run_op("cross_entropy", [xs, ls], [((1,), F32), ((T, Vp), dt)], attrs)]
    xi = xs.clone()
    loss = torch.empty(1, device=xi.device, dtype=torch.float32)
    run_op("cross_entropy", [xi, ls], [((1,), F32), ((T, Vp), dt)], attrs, outs=[loss, xi])
    torch.cuda.synchronize()
    assert bits_equal(from_torch(loss), sep[0]) and bits_equal(from_torch(xi), sep[1])


def test_unimplemented_is_loud():
    from paper_2303_04759_b200.runtime import Plan, UnimplementedOp
    with pytest.raises(UnimplementedOp):
        Plan("b200.no_such_op", [((4,), F32)], [((4,), F32)])
    with pytest.raises(UnimplementedOp):
        Plan("ref.add", [((4,), F32), ((4,), F32)], [((4,), F32)])


@pytest.mark.parametrize("H", [768, 100])
def test_embedding_sum_bit_exact(H):
    """embedding_sum (word + position + token type, rounded after each add)
    equals the oracle's chain bit for bit; H=100 takes the scalar path."""
    T = 300
    ids = [RNG.integers(0, v, size=T).astype(np.int32) for v in (1000, 512, 2)]
    tabs = [rn(v, H) for v in (1000, 512, 2)]
    ins = [(i, I32) for i in ids] + [(t, BF16) for t in tabs]
    g, o = run_both("embedding_sum", ins, [((T, H), BF16)])
    assert bits_equal(g[0], o[0])


def test_layer_norm_post_dropout_fused():
    """Embedding LayerNorm with its output dropout folded in (layer_norm
    post_dropout) and the backward's incoming-gradient dropout folded into
    layer_norm_dx (in_p): bit-identical to the separate dropout ops."""
    T, H = 300, 768
    x, gm, bt = rn(T, H), rn(H, lo=0.5, hi=1.5), rn(H, lo=-0.1, hi=0.1)
    dat = {"p": 0.1, "seed": 21, "salt": 3}
    outs = [((T, H), BF16), ((T,), F32), ((T,), F32)]
    g, o = run_both("layer_norm", [(x, BF16), (gm, BF16), (bt, BF16)], outs, {"eps": 1e-12, "post_dropout": 1, **dat})
    g0, _ = run_both("layer_norm", [(x, BF16), (gm, BF16), (bt, BF16)], outs, {"eps": 1e-12})
    gd, _ = run_both("dropout", [(g0[0], BF16)], [((T, H), BF16)], dat)
    assert bits_equal(g[0], gd[0]) and bits_equal(g[1], g0[1])
    assert rel_err(g[0], o[0]) < BF16_TOL
    dy = rn(T, H)
    ins = [(x, BF16), (gm, BF16), (g[1], F32), (g[2], F32)]
    lo = [((T, H), BF16), ((H,), F32), ((H,), F32)]
    gf, of = run_both("layer_norm_dx", ins + [(dy, BF16)], lo, {"in_p": 0.1, "in_seed": 21, "in_salt": 3})
    dd, _ = run_both("dropout", [(dy, BF16)], [((T, H), BF16)], dat)
    gu, _ = run_both("layer_norm_dx", ins + [(dd[0], BF16)], lo, {})
    for a, b in zip(gf, gu):
        assert bits_equal(a, b)
    assert rel_err(gf[0], of[0]) < 5e-3 and rel_err(gf[1], of[1]) < 1e-5
