"""Pin the CPU oracle (oracle/oracle.c) against the reference itself.

oracle/_ref/libtrainc_ref.so is the reference's exec_base compiled from
/root/reference/proj/include (oracle/Makefile).  Every base op the reference
implements must agree BIT FOR BIT with the restatement on seeded inputs, plus the
SPEC.md known answers.  These run on CPU.
"""
import numpy as np
import pytest

from oracle import oracle_py as O
from oracle.oracle_py import F16, F32, I32

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def rnd(seed, shape, lo=-1.0, hi=1.0, f16=False):
    n = int(np.prod(shape))
    x = O.rng_uniform(seed, n, lo, hi).reshape(shape)
    if f16:
        x = np.array([O.lib().orc_quantize_f16(float(v)) for v in x.ravel()],
                     dtype=np.float32).reshape(shape)
    return x


def both(op, inputs, out_specs, attrs=None):
    a = O.run(op, inputs, out_specs, attrs, impl="oracle")
    b = O.run(op, inputs, out_specs, attrs, impl="ref")
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), f"{op} not bit-exact"
    return a


# --- rng and rounding ---------------------------------------------------------

@needs_ref
def test_rng_matches_reference_mt19937():
    for seed in (0, 1, 42, 1234, 2**40 + 7):
        assert np.array_equal(O.rng_uniform(seed, 5000, -0.02, 0.02),
                              O.rng_uniform(seed, 5000, -0.02, 0.02, impl="ref"))
        assert np.array_equal(O.rng_below(seed, 5000, 30522),
                              O.rng_below(seed, 5000, 30522, impl="ref"))


@needs_ref
def test_f16_all_65536_patterns():
    """cast_f16 is exactly RNE on all 65,536 patterns."""
    L, R = O.lib(), O.ref()
    for h in range(65536):
        f = R.ref_half_bits_to_float(h)
        assert np.float32(L.orc_half_bits_to_float(h)).view(np.uint32) == np.float32(f).view(np.uint32) \
            or (np.isnan(f) and np.isnan(L.orc_half_bits_to_float(h)))
        if not np.isnan(f):
            assert L.orc_float_to_half_bits(f) == R.ref_float_to_half_bits(f) == h or \
                (h == 0x8000 and f == 0.0)


@needs_ref
def test_f16_rounding_random_floats():
    L, R = O.lib(), O.ref()
    xs = np.concatenate([O.rng_uniform(3, 20000, -70000.0, 70000.0),
                         O.rng_uniform(4, 20000, -1e-4, 1e-4),
                         O.rng_uniform(5, 5000, -1e-7, 1e-7)])
    for f in xs:
        assert L.orc_float_to_half_bits(float(f)) == R.ref_float_to_half_bits(float(f))


def test_bf16_rounding_rne():
    L = O.lib()
    # halfway cases: 1 + 2^-8 is exactly between two bf16 values -> even (1.0)
    assert L.orc_quantize_bf16(1.0 + 2.0 ** -8) == 1.0
    assert L.orc_quantize_bf16(1.0 + 3 * 2.0 ** -8) == 1.0 + 2.0 ** -6
    from paper_2303_04759_b200.abi import bf16_round
    xs = O.rng_uniform(9, 10000, -1000.0, 1000.0)
    ours = np.array([L.orc_quantize_bf16(float(v)) for v in xs], dtype=np.float32)
    assert np.array_equal(ours, bf16_round(xs))


# --- elementwise (backends.hpp:67-93,168-177) -----------------------------------

@needs_ref
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "tanh_dx"])
@pytest.mark.parametrize("f16", [False, True])
def test_binary_ops_bit_exact(op, f16):
    d = F16 if f16 else F32
    a = O.HostTensor(rnd(1, (6, 7), f16=f16), d)
    b = O.HostTensor(rnd(2, (6, 7), 0.5, 2.0, f16=f16), d)
    both(op, [a, b], [((6, 7), d)])
    # broadcasts: trailing dim, scalar b, scalar a, and size-1 pinning
    both(op, [a, O.HostTensor(rnd(3, (7,), f16=f16), d)], [((6, 7), d)])
    both(op, [a, O.HostTensor(np.array([0.75], np.float32), d)], [((6, 7), d)])
    both(op, [O.HostTensor(np.array([1.5], np.float32), d), b], [((6, 7), d)])
    both(op, [O.HostTensor(rnd(4, (6, 1), f16=f16), d), O.HostTensor(rnd(5, (1, 7), 0.5, 1.5, f16=f16), d)],
         [((6, 7), d)])
    both(op, [O.HostTensor(rnd(6, (2, 3, 4), f16=f16), d), O.HostTensor(rnd(7, (3, 1), 0.5, 1.5, f16=f16), d)],
         [((2, 3, 4), d)])


@needs_ref
@pytest.mark.parametrize("op", ["neg", "tanh", "relu", "gtz"])
@pytest.mark.parametrize("f16", [False, True])
def test_unary_ops_bit_exact(op, f16):
    d = F16 if f16 else F32
    x = O.HostTensor(rnd(11, (5, 9), -3, 3, f16=f16), d)
    both(op, [x], [((5, 9), d)])


def test_spec_known_answers():
    """relu(-1)=0; matmul(M,I)=M; sum([.1,.2,.3]) = left fold."""
    assert O.run("relu", [np.array([-1.0], np.float32)], [((1,), F32)])[0][0] == 0.0
    m = rnd(21, (4, 4))
    eye = np.eye(4, dtype=np.float32)
    assert np.array_equal(O.run("matmul", [m, eye], [((4, 4), F32)])[0], m)
    s = O.run("sum", [np.array([0.1, 0.2, 0.3], np.float32)], [((1,), F32)])[0][0]
    assert s == (np.float32(0.1) + np.float32(0.2)) + np.float32(0.3)


# --- cast / bcast / transpose / reshape ----------------------------------------

@needs_ref
def test_layout_ops_bit_exact():
    x = O.HostTensor(rnd(31, (4, 6), -9, 9), F32)
    both("cast", [x], [((4, 6), F16)], {"to": "f16"})
    both("cast", [x], [((4, 6), F32)], {"to": "f32"})
    both("bcast", [O.HostTensor(rnd(32, (6,)), F32)], [((3, 4, 6), F32)], {"shape": "3,4,6"})
    both("transpose", [x], [((6, 4), F32)])
    both("reshape", [x], [((2, 12), F32)], {"shape": "2,12"})


# --- reductions (backends.hpp:95-141) -------------------------------------------

@needs_ref
@pytest.mark.parametrize("op", ["sum", "mean"])
def test_reductions_bit_exact(op):
    x = O.HostTensor(rnd(41, (3, 5, 7), -2, 2), F32)
    both(op, [x], [((1,), F32)])
    both(op, [x], [((5, 7), F32)], {"axes": "0"})
    both(op, [x], [((3, 7), F32)], {"axes": "1"})
    both(op, [x], [((3, 5), F32)], {"axes": "2"})
    both(op, [x], [((5,), F32)], {"axes": "0,2"})
    both(op, [x], [((3, 1, 7), F32)], {"axes": "1", "keepdims": 1})
    xh = O.HostTensor(rnd(42, (8, 16), -2, 2, f16=True), F16)
    both(op, [xh], [((16,), F16)], {"axes": "0"})


@needs_ref
def test_mse_bit_exact():
    both("mse", [rnd(51, (9, 4)), rnd(52, (9, 4))], [((1,), F32)])


# --- matmul (backends.hpp:143-155, 280-324) --------------------------------------

@needs_ref
@pytest.mark.parametrize("mnk", [(2, 4, 3), (33, 33, 33), (64, 48, 80)])
def test_matmul_bit_exact(mnk):
    m, n, k = mnk
    a, b = rnd(61, (m, k)), rnd(62, (k, n))
    out = both("matmul", [a, b], [((m, n), F32)])[0]
    # opt.matmul (blocked, tile 32) has the same per-element k order
    import ctypes
    A, B, C = O.HostTensor(a), O.HostTensor(b), O.HostTensor(np.zeros((m, n), np.float32))
    assert O.ref().ref_exec_opt(ctypes.byref(A.desc()), ctypes.byref(B.desc()), None, 0,
                                ctypes.byref(C.desc())) == 0
    assert np.array_equal(C.arr, out)


@needs_ref
@pytest.mark.parametrize("act,name", [(0, "none"), (1, "relu"), (2, "tanh")])
def test_linear_matches_matmul_add_act(act, name):
    """oracle `linear` == opt-dialect matmul_add_act (backends.hpp:311-324)."""
    import ctypes
    m, n, k = 17, 12, 9
    a, b, bias = rnd(71, (m, k)), rnd(72, (k, n)), rnd(73, (n,))
    ours = O.run("linear", [a, b, bias], [((m, n), F32)], {"act": name})[0]
    A, B, Bi = O.HostTensor(a), O.HostTensor(b), O.HostTensor(bias)
    C = O.HostTensor(np.zeros((m, n), np.float32))
    assert O.ref().ref_exec_opt(ctypes.byref(A.desc()), ctypes.byref(B.desc()),
                                ctypes.byref(Bi.desc()), act, ctypes.byref(C.desc())) == 0
    assert np.array_equal(C.arr.view(np.uint32), ours.view(np.uint32))


# --- optimizers ----------------------------------------------------------------

@needs_ref
def test_sgd_bit_exact():
    both("sgd_update", [rnd(81, (10, 3)), rnd(82, (10, 3))], [((10, 3), F32)], {"lr": 0.01})


@needs_ref
@pytest.mark.parametrize("t", [1.0, 2.0, 17.0])
def test_adam_bit_exact(t):
    p, g = rnd(91, (50,)), rnd(92, (50,))
    m, v = rnd(93, (50,), -0.1, 0.1), rnd(94, (50,), 0.0, 0.01)
    attrs = {"lr": 1e-3, "beta1": 0.9, "beta2": 0.999, "eps": 1e-6}
    both("adam_update", [p, g, m, v, np.array([t], np.float32)], [((50,), F32)] * 3, attrs)


# --- collectives at world 1 (backends.hpp:245-273) --------------------------------

@needs_ref
def test_world1_collectives_bit_exact():
    x = rnd(101, (2, 5))
    both("allreduce", [x], [((2, 5), F32)], {"world": 1})
    both("reduce_scatter", [x], [((10,), F32)], {"world": 1})
    both("all_gather", [rnd(102, (10,))], [((2, 5), F32)], {"world": 1, "shape": "2,5"})
    both("shard", [x], [((10,), F32)], {"world": 1})
    both("reduce_scatter_batched", [x, rnd(103, (3,))], [((10,), F32), ((3,), F32)], {"world": 1})


def test_world_gt1_requires_bus():
    with pytest.raises(RuntimeError, match="simulation bus"):
        O.run("allreduce", [rnd(1, (4,))], [((4,), F32)], {"world": 2})
    if O.ref_available():
        with pytest.raises(RuntimeError, match="simulation bus"):
            O.run("allreduce", [rnd(1, (4,))], [((4,), F32)], {"world": 2}, impl="ref")
