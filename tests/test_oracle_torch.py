"""Independent check of the oracle's EXTENSION ops (the transformer ops the
reference does not have -- SURVEY.md §2.4 / §8c "parity unpinned by the
reference"): every oracle.c kernel for them is compared against PyTorch on the
CPU in float64, forward values and -- for the `_dx` ops -- the gradients torch
autograd derives from the forward definition.  torch is an independent
implementation of the same mathematics (its LayerNorm, softmax, GELU(erf),
cross-entropy with ignore_index, scatter-add), so a semantic slip in oracle.c
(a wrong adjoint, a mis-scaled dropout, a mis-indexed head) fails here even
though the device kernels are written against that oracle.

Inputs are f32 (the oracle's exec_base dtype); tolerance 1e-5 norm-wise for
forward values, 1e-4 for gradients (f32 vs f64 accumulation), over several
seeds and ragged shapes.  CPU only.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle_py as O  # noqa: E402
from paper_2303_04759_b200.abi import F32, I32  # noqa: E402

SEEDS = [0, 1, 2, 3, 4]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rn(rng, *shape, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, shape).astype(np.float32)


def t64(a, grad=False):
    t = torch.from_numpy(np.asarray(a, np.float64).copy())
    t.requires_grad_(grad)
    return t


# ---------------------------------------------------------------- LayerNorm
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("T,H", [(7, 32), (33, 100)])
def test_layer_norm_fwd_bwd_vs_torch(seed, T, H):
    rng = np.random.default_rng(seed)
    x, g, b, dy = rn(rng, T, H, lo=-3, hi=3), rn(rng, H, lo=0.5, hi=1.5), rn(rng, H), rn(rng, T, H)
    eps = 1e-5
    y, mean, rstd = O.run("layer_norm", [x, g, b], [((T, H), F32), ((T,), F32), ((T,), F32)], {"eps": eps})
    xt, gt, bt = t64(x, True), t64(g, True), t64(b, True)
    yt = torch.nn.functional.layer_norm(xt, (H,), gt, bt, eps)
    assert rel(y, yt.detach()) < 1e-5
    assert rel(mean, xt.detach().mean(1)) < 1e-5
    assert rel(rstd, 1 / torch.sqrt(xt.detach().var(1, unbiased=False) + eps)) < 1e-5
    yt.backward(t64(dy))
    dx, dg, db = O.run("layer_norm_dx", [x, g, mean, rstd, dy], [((T, H), F32), ((H,), F32), ((H,), F32)])
    assert rel(dx, xt.grad) < 1e-4
    assert rel(dg, gt.grad) < 1e-4
    assert rel(db, bt.grad) < 1e-4


@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("p", [0.0, 0.2])
def test_add_layer_norm_dropout_residual_vs_torch(seed, p):
    """add_layer_norm(x, r): s = dropout(x) + r, y = LN(s); layer_norm_dx with
    a second incoming gradient dy2 at y (fan-out of the residual stream) and dx =
    dropout'(ds) -- against torch autograd of the same composition with the
    same keep mask."""
    rng = np.random.default_rng(seed)
    T, H = 9, 48
    x, r = rn(rng, T, H), rn(rng, T, H)
    g, b = rn(rng, H, lo=0.5, hi=1.5), rn(rng, H)
    dy, dy2 = rn(rng, T, H), rn(rng, T, H)
    at = {"eps": 1e-12, "p": p, "seed": 7 + seed, "salt": 3}
    y, s, mean, rstd = O.run("add_layer_norm", [x, r, g, b],
                             [((T, H), F32), ((T, H), F32), ((T,), F32), ((T,), F32)], at)
    keep = O.dropout_keep_mask(7 + seed, 3, T * H, p).reshape(T, H).astype(np.float64)
    xt, rt, gt, bt = t64(x, True), t64(r, True), t64(g, True), t64(b, True)
    st = xt * t64(keep) / (1.0 - p) + rt
    yt = torch.nn.functional.layer_norm(st, (H,), gt, bt, 1e-12)
    assert rel(s, st.detach()) < 1e-6
    assert rel(y, yt.detach()) < 1e-5
    # y fans out (next sublayer + the residual path): both gradients arrive at y
    yt.backward(t64(dy) + t64(dy2))
    ds, dg, db, dx = O.run("layer_norm_dx", [s, g, mean, rstd, dy, dy2],
                           [((T, H), F32), ((H,), F32), ((H,), F32), ((T, H), F32)], at)
    assert rel(ds, rt.grad) < 1e-4  # r's gradient is ds itself
    assert rel(dx, xt.grad) < 1e-4
    assert rel(dg, gt.grad) < 1e-4 and rel(db, bt.grad) < 1e-4


# --------------------------------------------------------------------- GELU
@pytest.mark.parametrize("seed", SEEDS)
def test_gelu_and_dx_vs_torch(seed):
    rng = np.random.default_rng(seed)
    x, dy = rn(rng, 1000, lo=-6, hi=6), rn(rng, 1000)
    (y,) = O.run("gelu", [x], [((1000,), F32)])
    xt = t64(x, True)
    yt = torch.nn.functional.gelu(xt)  # exact (erf) GELU
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-6
    yt.backward(t64(dy))
    (dx,) = O.run("gelu_dx", [x, dy], [((1000,), F32)])
    assert rel(dx, xt.grad) < 1e-5


@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("act", ["gelu", "relu", "tanh"])
def test_linear_act_saved_derivative_vs_torch(seed, act):
    """y = act(x W1 + b1) (linear), z = y W2.  linear(save=grad) stores
    act'(u); the backward's fused dgrad matmul_dact(dz, W2^T, act'(u),
    act=deriv) must equal dL/du, and matmul_dact on the saved pre-activation
    (save=preact, act=<act>) the same -- against torch autograd."""
    rng = np.random.default_rng(seed)
    M, K, N, N2 = 13, 24, 17, 9
    x, w, b, w2, dz = rn(rng, M, K), rn(rng, K, N), rn(rng, N), rn(rng, N, N2), rn(rng, M, N2)
    y, d = O.run("linear", [x, w, b], [((M, N), F32), ((M, N), F32)],
                 {"act": act, "save_preact": 1, "save": "grad"})
    _, u = O.run("linear", [x, w, b], [((M, N), F32), ((M, N), F32)], {"act": act, "save_preact": 1})
    xt, wt, bt = t64(x, True), t64(w, True), t64(b, True)
    ut = xt @ wt + bt
    ut.retain_grad()
    f = {"gelu": torch.nn.functional.gelu, "relu": torch.relu, "tanh": torch.tanh}[act]
    yt = f(ut)
    assert rel(y, yt.detach()) < 1e-5
    assert rel(u, ut.detach()) < 1e-6
    (yt @ t64(w2)).backward(t64(dz))
    (du,) = O.run("matmul_dact", [dz, w2, d], [((M, N), F32)], {"act": "deriv", "tb": 1})
    assert rel(du, ut.grad) < 1e-5
    if act != "tanh":  # tanh's aux is its output y (tanh_dx semantics), not u
        (du2,) = O.run("matmul_dact", [dz, w2, u], [((M, N), F32)], {"act": act, "tb": 1})
        assert rel(du2, ut.grad) < 1e-5
    else:
        (du2,) = O.run("matmul_dact", [dz, w2, y], [((M, N), F32)], {"act": act, "tb": 1})
        assert rel(du2, ut.grad) < 1e-5
    (dx,) = O.run("matmul_t", [du, w], [((M, K), F32)], {"tb": 1})
    assert rel(dx, xt.grad) < 1e-5
    (dw,) = O.run("matmul_t", [x, du], [((K, N), F32)], {"ta": 1})
    assert rel(dw, wt.grad) < 1e-5
    (dbias,) = O.run("colsum", [du], [((N,), F32)])
    assert rel(dbias, bt.grad) < 1e-5


# ------------------------------------------------------------------ softmax
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("causal", [0, 1])
def test_softmax_and_dx_vs_torch(seed, causal):
    rng = np.random.default_rng(seed)
    Z, S = 3, 11
    x, dy = rn(rng, Z, S, S, lo=-4, hi=4), rn(rng, Z, S, S)
    scale = 0.37
    (y,) = O.run("softmax", [x], [((Z, S, S), F32)], {"scale": scale, "causal": causal})
    xt = t64(x, True)
    v = xt * scale
    if causal:
        v = v.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
    yt = torch.softmax(v, -1)
    assert rel(y, yt.detach()) < 1e-6
    yt.backward(t64(dy))
    (dx,) = O.run("softmax_dx", [y, dy], [((Z, S, S), F32)], {"scale": scale})
    assert rel(dx, xt.grad) < 1e-5


# ---------------------------------------------------------------- attention
def torch_attention(qkv, B, S, A, p, keep, causal):
    """qkv [B*S, 3H] packed (q | k | v), heads of width dh inside each third."""
    H = qkv.shape[1] // 3
    dh = H // A
    q, k, v = qkv[:, :H], qkv[:, H:2 * H], qkv[:, 2 * H:]
    sh = lambda t: t.reshape(B, S, A, dh).permute(0, 2, 1, 3)  # noqa: E731
    s = sh(q) @ sh(k).transpose(-1, -2) / np.sqrt(dh)
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
    P = torch.softmax(s, -1)
    Pd = P * keep / (1.0 - p) if p > 0 else P
    ctx = (Pd @ sh(v)).permute(0, 2, 1, 3).reshape(B * S, H)
    return ctx, P.reshape(B * A * S, S)


@pytest.mark.parametrize("seed", SEEDS[:3])
@pytest.mark.parametrize("p,causal", [(0.0, 0), (0.25, 0), (0.0, 1), (0.25, 1)])
def test_attention_fwd_bwd_vs_torch(seed, p, causal):
    rng = np.random.default_rng(seed)
    B, S, A, dh = 2, 12, 3, 8
    H, T = A * dh, B * S
    qkv, dctx = rn(rng, T, 3 * H, lo=-2, hi=2), rn(rng, T, H)
    at = {"heads": A, "seq": S, "p": p, "seed": 21 + seed, "salt": 4, "causal": causal}
    ctx, probs = O.run("attention", [qkv], [((T, H), F32), ((B * A * S, S), F32)], at)
    # keep bit of element (z, i, j): Philox index (z*S + i)*S + j
    keep = O.dropout_keep_mask(21 + seed, 4, B * A * S * S, p).reshape(B, A, S, S).astype(np.float64)
    qt = t64(qkv, True)
    ct, pt = torch_attention(qt, B, S, A, p, t64(keep), causal)
    assert rel(probs, pt.detach()) < 1e-5
    assert rel(ctx, ct.detach()) < 1e-5
    ct.backward(t64(dctx))
    (dqkv,) = O.run("attention_dx", [qkv, probs, dctx], [((T, 3 * H), F32)], at)
    assert rel(dqkv, qt.grad) < 1e-4


# ------------------------------------------------------------ cross entropy
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("gscale", [1.0, 0.5])
def test_cross_entropy_ignore_index_padding_vs_torch(seed, gscale):
    """loss = mean over labelled rows of (lse - x[label]) over the first
    `classes` columns; padded columns get zero gradient; ignored rows (-100)
    contribute nothing -- torch F.cross_entropy(ignore_index=-100)."""
    rng = np.random.default_rng(seed)
    T, V, Vp = 20, 37, 64
    x = rn(rng, T, Vp, lo=-5, hi=5)
    lab = rng.integers(0, V, T).astype(np.int32)
    lab[rng.random(T) < 0.4] = -100
    lab[0] = 3
    loss, dl = O.run("cross_entropy", [x, O.HostTensor(lab, I32)], [((1,), F32), ((T, Vp), F32)],
                     {"classes": V, "ignore_index": -100, "grad": 1, "grad_scale": gscale})
    xt = t64(x[:, :V], True)
    lt = torch.nn.functional.cross_entropy(xt, torch.from_numpy(lab.astype(np.int64)), ignore_index=-100)
    assert abs(float(loss[0]) - lt.item()) <= 1e-5 * abs(lt.item())
    (lt * gscale).backward()
    assert rel(dl[:, :V], xt.grad) < 1e-5
    assert not np.any(dl[:, V:])


# ---------------------------------------------------------------- embedding
@pytest.mark.parametrize("seed", SEEDS)
def test_embedding_gather_scatter_vs_torch(seed):
    rng = np.random.default_rng(seed)
    T, V, H = 50, 13, 8  # many repeated ids -> collisions in the scatter-add
    ids = rng.integers(0, V, T).astype(np.int32)
    tab, dy, base = rn(rng, V, H), rn(rng, T, H), rn(rng, V, H)
    (e,) = O.run("embedding", [O.HostTensor(ids, I32), tab], [((T, H), F32)])
    tt = t64(tab, True)
    et = torch.nn.functional.embedding(torch.from_numpy(ids.astype(np.int64)), tt)
    assert np.array_equal(e, et.detach().numpy().astype(np.float32))
    et.backward(t64(dy))
    (d0,) = O.run("embedding_dx", [O.HostTensor(ids, I32), dy], [((V, H), F32)])
    assert rel(d0, tt.grad) < 1e-6
    (d1,) = O.run("embedding_dx", [O.HostTensor(ids, I32), dy, base], [((V, H), F32)])
    assert rel(d1, tt.grad + t64(base)) < 1e-6


@pytest.mark.parametrize("seed", SEEDS)
def test_embedding_sum_vs_torch(seed):
    rng = np.random.default_rng(seed)
    T, H = 16, 8
    ids = [rng.integers(0, n, T).astype(np.int32) for n in (11, 6, 2)]
    tabs = [rn(rng, n, H) for n in (11, 6, 2)]
    (e,) = O.run("embedding_sum", [O.HostTensor(i, I32) for i in ids] + tabs, [((T, H), F32)])
    ref = sum(t64(t)[torch.from_numpy(i.astype(np.int64))] for i, t in zip(ids, tabs))
    assert rel(e, ref) < 1e-6


# ------------------------------------------------------------------ dropout
@pytest.mark.parametrize("p", [0.1, 0.5])
def test_dropout_rate_and_scale(p):
    """dropout keeps each element with probability 1 - p (Philox, 16-bit
    draws) and scales kept values by 1/(1-p); the empirical keep rate over
    2^16 elements is within 4 sigma of 1 - p."""
    n = 1 << 16
    x = np.ones(n, np.float32)
    (y,) = O.run("dropout", [x], [((n,), F32)], {"p": p, "seed": 9, "salt": 2})
    kept = y != 0
    assert np.allclose(y[kept], np.float32(1.0 / (1.0 - p)))
    rate = kept.mean()
    sigma = np.sqrt(p * (1 - p) / n)
    assert abs(rate - (1 - p)) < 4 * sigma, rate


@pytest.mark.parametrize("seed", SEEDS[:3])
@pytest.mark.parametrize("p,causal,S", [(0.0, 0, 12), (0.25, 0, 12), (0.0, 1, 40), (0.25, 1, 40)])
def test_attention_lse_fwd_bwd_vs_torch(seed, p, causal, S):
    """attention lse=1 (the flash formulation): ctx and the per-row
    log-sum-exp vs torch; attention_dx(qkv, ctx, lse, dctx) vs torch autograd
    (f32: the dS / Pd roundings are identities)."""
    rng = np.random.default_rng(seed)
    B, A, dh = 2, 3, 8
    H, T = A * dh, B * S
    qkv, dctx = rn(rng, T, 3 * H, lo=-2, hi=2), rn(rng, T, H)
    at = {"heads": A, "seq": S, "p": p, "seed": 21 + seed, "salt": 4, "causal": causal, "lse": 1}
    ctx, lse = O.run("attention", [qkv], [((T, H), F32), ((B * A * S,), F32)], at)
    keep = O.dropout_keep_mask(21 + seed, 4, B * A * S * S, p).reshape(B, A, S, S).astype(np.float64)
    qt = t64(qkv, True)
    ct, pt = torch_attention(qt, B, S, A, p, t64(keep), causal)
    assert rel(ctx, ct.detach()) < 1e-5
    q_, k_ = qt.detach()[:, :H], qt.detach()[:, H:2 * H]
    sh = lambda t: t.reshape(B, S, A, dh).permute(0, 2, 1, 3)  # noqa: E731
    sc = sh(q_) @ sh(k_).transpose(-1, -2) / np.sqrt(dh)
    if causal:
        sc = sc.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
    assert rel(lse, torch.logsumexp(sc, -1).reshape(-1)) < 1e-6
    ct.backward(t64(dctx))
    (dqkv,) = O.run("attention_dx", [qkv, ctx, lse, dctx], [((T, 3 * H), F32)], at)
    # D uses the stored (f32) ctx: exact here
    assert rel(dqkv, qt.grad) < 1e-4, rel(dqkv, qt.grad)
