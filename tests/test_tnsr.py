"""TNSR tensor files (tensor.hpp:76-139) and checkpoint/resume of the step state.

CPU tests pin three implementations against each other on the same tensors:
the reference's own save_tensor/load_tensor (oracle/_ref), the numpy
restatement (oracle_py.tnsr_*), and the product's native reader/writer
(host/tnsr.hpp through libtrainc_b200.so).  f32/f16 files must be
byte-identical in both directions; bf16 (code 2) and i32 (code 3) are the
backend's extension and round-trip bit-exactly.  The GPU test checkpoints a
bf16 + Adam BERT session after two steps, restores it into a fresh session and
requires the next step's loss and state to be bit-identical to the
uninterrupted run.
"""
import os

import numpy as np
import pytest

from oracle import oracle_py as O
from paper_2303_04759_b200 import session as S

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

SHAPES = [(), (1,), (7,), (3, 5), (2, 3, 4), (2, 1, 3, 1, 2)]


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape).astype(np.float32) * 10.0


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


@needs_ref
@pytest.mark.parametrize("shape", SHAPES)
def test_f32_bytes_match_reference(tmp_path, shape):
    x = _rand(shape, 1)
    O.ref_tnsr_save(str(tmp_path / "ref.tnsr"), x, 0)
    S.tnsr_save(str(tmp_path / "ours.tnsr"), x)
    ref = _bytes(tmp_path / "ref.tnsr")
    assert _bytes(tmp_path / "ours.tnsr") == ref
    assert O.tnsr_bytes(x, 0) == ref
    y, code = S.tnsr_load(str(tmp_path / "ref.tnsr"))
    assert code == 0 and y.shape == x.shape and np.array_equal(y.view(np.uint32), x.view(np.uint32))


@needs_ref
@pytest.mark.parametrize("shape", SHAPES)
def test_f16_bytes_match_reference(tmp_path, shape):
    # the reference rounds floats to f16 on save (float_to_half_bits, RNE); hand
    # it values that are already f16 so both sides store the same bits
    x16 = _rand(shape, 2).astype(np.float16)
    O.ref_tnsr_save(str(tmp_path / "ref.tnsr"), x16.astype(np.float32), 1)
    S.tnsr_save(str(tmp_path / "ours.tnsr"), x16)
    ref = _bytes(tmp_path / "ref.tnsr")
    assert _bytes(tmp_path / "ours.tnsr") == ref
    assert O.tnsr_bytes(x16, 1) == ref
    # the reference's loader reads our file and widens exactly
    y, code = O.ref_tnsr_load(str(tmp_path / "ours.tnsr"), max(x16.size, 1))
    assert code == 1 and y.shape == x16.shape
    assert np.array_equal(y, x16.astype(np.float32))


@needs_ref
def test_reference_f16_rounding_matches_numpy(tmp_path):
    """Unrounded floats: the reference's RNE on save equals numpy's f16 cast,
    including subnormals, overflow to inf and ties."""
    x = np.concatenate([_rand((4096,), 3), np.array([65520.0, 65504.0, 1e-7, 6e-8, -3e-5, 2049.0, 2051.0],
                                                    np.float32)])
    O.ref_tnsr_save(str(tmp_path / "ref.tnsr"), x, 1)
    y, code = S.tnsr_load(str(tmp_path / "ref.tnsr"))
    assert code == 1
    assert np.array_equal(y.view(np.uint16), x.astype(np.float16).view(np.uint16))


@needs_ref
def test_reference_reads_our_f32(tmp_path):
    x = _rand((4, 6), 4)
    S.tnsr_save(str(tmp_path / "ours.tnsr"), x)
    y, code = O.ref_tnsr_load(str(tmp_path / "ours.tnsr"), x.size)
    assert code == 0 and np.array_equal(y, x)


@pytest.mark.parametrize("code,dtype", [(2, np.uint16), (3, np.int32)])
def test_extension_codes_round_trip(tmp_path, code, dtype):
    rng = np.random.default_rng(5)
    x = rng.integers(np.iinfo(dtype).min, np.iinfo(dtype).max, (3, 17), dtype=dtype, endpoint=True)
    S.tnsr_save(str(tmp_path / "x.tnsr"), x, code)
    assert _bytes(tmp_path / "x.tnsr") == O.tnsr_bytes(x, code)
    y, c = S.tnsr_load(str(tmp_path / "x.tnsr"))
    assert c == code and y.dtype == dtype and np.array_equal(y, x)
    z, c2 = O.tnsr_parse(_bytes(tmp_path / "x.tnsr"))
    assert c2 == code and np.array_equal(z, x)


@needs_ref
def test_reference_rejects_extension_codes(tmp_path):
    """Files with the bf16/i32 codes are outside the reference's format: its
    loader refuses them with its header error (no silent misread)."""
    S.tnsr_save(str(tmp_path / "b.tnsr"), np.zeros(4, np.uint16), 2)
    with pytest.raises(RuntimeError, match="bad tensor file header"):
        O.ref_tnsr_load(str(tmp_path / "b.tnsr"), 4)


def test_errors_match_reference_messages(tmp_path):
    p = str(tmp_path / "bad.tnsr")
    with open(p, "wb") as f:
        f.write(b"TNSX\x00\x01" + bytes(8))
    with pytest.raises(RuntimeError, match="bad tensor file magic"):
        S.tnsr_load(p)
    with open(p, "wb") as f:
        f.write(b"TNSR\x07\x01" + bytes(8))
    with pytest.raises(RuntimeError, match="bad tensor file header"):
        S.tnsr_load(p)
    full = O.tnsr_bytes(np.arange(10, dtype=np.float32), 0)
    with open(p, "wb") as f:
        f.write(full[:-3])
    with pytest.raises(RuntimeError, match="truncated tensor file"):
        S.tnsr_load(p)
    with open(p, "wb") as f:
        f.write(full[:9])  # inside the dims
    with pytest.raises(RuntimeError, match="truncated tensor file"):
        S.tnsr_load(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        S.tnsr_load(str(tmp_path / "missing" / "x.tnsr"))
    with pytest.raises(RuntimeError, match="cannot open"):
        S.tnsr_save(str(tmp_path / "missing" / "x.tnsr"), np.zeros(2, np.float32))


def test_native_load_size_check(tmp_path):
    p = str(tmp_path / "x.tnsr")
    S.tnsr_save(p, np.zeros((2, 3), np.float32))
    buf = np.empty(5, np.float32)
    rc = S.lib().tb_tnsr_load(os.fsencode(p), buf.ctypes.data, buf.nbytes)
    assert rc != 0 and "size mismatch" in S.lib().tb_last_error().decode()


@pytest.mark.gpu
def test_checkpoint_resume_bit_identical(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = S.ModelConfig.tiny(dtype="bf16", opt="adam", lr=1e-3, L=2, B=4)
    batches = [S.synthetic_batch(cfg, seed=cfg.seed_d + k) for k in range(3)]

    a = S.Session(cfg)
    a.init_params()
    for ids, labels in batches[:2]:
        a.set_batch(ids, labels)
        a.step()
    names = a.save_checkpoint(str(tmp_path / "ck"))
    assert set(names) == {"params", "p16", "m", "v", "step"}
    a.set_batch(*batches[2])
    a.step()
    loss_a = a.loss()
    state_a = {n: a.read(n, np.uint16 if n == "p16" else np.float32) for n in names}

    b = S.Session(cfg)  # fresh session, never initialised: all state comes from the files
    b.load_checkpoint(str(tmp_path / "ck"))
    b.set_batch(*batches[2])
    b.step()
    loss_b = b.loss()
    assert np.float32(loss_a).tobytes() == np.float32(loss_b).tobytes()
    for n in names:
        got = b.read(n, np.uint16 if n == "p16" else np.float32)
        assert np.array_equal(got.view(np.uint8), state_a[n].view(np.uint8)), n

    # the checkpoint files are plain TNSR: master weights read back as f32,
    # the compute copy as bf16 (code 2)
    p, code = S.tnsr_load(str(tmp_path / "ck" / "params.tnsr"))
    assert code == 0 and p.dtype == np.float32
    p16, code16 = S.tnsr_load(str(tmp_path / "ck" / "p16.tnsr"))
    assert code16 == 2 and p16.dtype == np.uint16

    # a file for a different graph is refused, not reinterpreted
    S.tnsr_save(str(tmp_path / "wrong.tnsr"), np.zeros(3, np.float32))
    with pytest.raises(RuntimeError, match="does not match parameter"):
        b.load_param("params", str(tmp_path / "wrong.tnsr"))
    a.close()
    b.close()


@pytest.mark.gpu
def test_train_report_csv_deterministic(tmp_path):
    """`trainc train --report`: header-only for 0 steps; the
    same seed twice gives identical CSVs except the timing column."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = S.ModelConfig.tiny(dtype="bf16", opt="adam", lr=1e-3)
    S.train_report(cfg, 0, str(tmp_path / "r0.csv"))
    assert open(tmp_path / "r0.csv").read() == "step,loss,iter_time,peak_pool_bytes\n"
    a = S.train_report(cfg, 5, str(tmp_path / "a.csv"), seed=11)
    b = S.train_report(cfg, 5, str(tmp_path / "b.csv"), seed=11)
    strip = lambda p: [l.split(",")[:2] + l.split(",")[3:] for l in open(p).read().splitlines()]
    assert strip(tmp_path / "a.csv") == strip(tmp_path / "b.csv")
    assert len(a) == 5 and all(r[2] > 0 for r in a) and all(r[3] > 0 for r in a)
