"""Kernel priority derivation from profiled medians (backends.hpp:387-419,
SPEC.md:618-625 "used by backends.derive_priorities"): the reference's own
derive_priorities, fed b200 device medians and the reference CPU dialects'
host medians for the same op and shape."""
import time

import numpy as np
import pytest

from paper_2303_04759_b200.session import derive_priorities


def test_derive_priorities_orders_by_median():
    pr = derive_priorities([("ref", "matmul", "64x64x64", 90.0), ("opt", "matmul", "64x64x64", 40.0),
                            ("b200", "matmul", "64x64x64", 4.0), ("ref", "add", "64", 1.0)])
    assert pr["b200.matmul"] > pr["opt.matmul"] > pr["ref.matmul"]
    assert pr == {"b200.matmul": 13, "opt.matmul": 12, "ref.matmul": 11, "ref.add": 11}


@pytest.mark.gpu
def test_profiled_b200_matmul_outranks_reference_dialects():
    """SPEC.md:624 example at 64x64x64: the b200 matmul's median device time
    (CUDA events over single launches) against the reference's ref (matmul_ref)
    and opt (matmul_blocked) kernels timed on the host; derive_priorities ranks
    b200 first and orders ref/opt by their measured medians."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from oracle import oracle_py as O
    from paper_2303_04759_b200.abi import F32
    from paper_2303_04759_b200.runtime import Plan
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    n = 64
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    plan = Plan("matmul_t", [((n, n), F32), ((n, n), F32)], [((n, n), F32)], {})
    s = torch.cuda.current_stream().cuda_stream
    meds = {}
    ts = []
    for _ in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch([a.data_ptr(), b.data_ptr()], [c.data_ptr()], s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    meds["b200"] = float(np.median(ts))
    an, bn = a.cpu().numpy(), b.cpu().numpy()
    for impl, fn in (("ref", lambda: O.run("matmul", [an, bn], [((n, n), F32)], impl="ref")),
                     ("opt", lambda: O.ref_opt_matmul(an, bn))):
        ts = []
        for _ in range(15):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e6)
        meds[impl] = float(np.median(ts))
    pr = derive_priorities([(d, "matmul", "64x64x64", us) for d, us in meds.items()])
    print("medians us", meds, "priorities", pr)
    assert pr["b200.matmul"] == max(pr.values())
    assert (pr["opt.matmul"] > pr["ref.matmul"]) == (meds["opt"] < meds["ref"])
