// k_gemm_ops.cu -- plan builders for the GEMM-shaped ops of the b200 dialect:
//   matmul        A[M,K].B[K,N]                        backends.hpp:143-155,215
//   matmul_t      alpha * op(A).op(B), out dtype attr   (absorbs `transpose` and
//                 `cast` into operand major-ness / epilogue)
//   linear        act(x.W + bias) [, pre-activation]    matmul_add_act, backends.hpp:311-324
//   matmul_dact   (op(A).op(B)) * act'(aux)             backward GEMM, fused dact
//   batch_matmul  rank-3 batched matmul_t
// f16/bf16 operands run on the tcgen05 kernel; f32 (or attr exact=1) runs the
// exact SIMT kernel, bit-identical to the reference.
#include "gemm.cuh"

namespace tcb {

// The reference dtypes (f32, emulated f16) keep the bit-exact contract of
// matmul_ref; bf16 (the AutoCast extension) runs on the tensor cores.
static bool want_exact(const Plan& p) {
  return p.in[0].dtype != TCB_BF16 || p.attrs.i("exact", 0) != 0;
}

// Fill the static part of a 2-D GEMM: A, B are rank-2 dense row-major.
static GemmArgs gemm2d(const Spec& A, const Spec& B, int ta, int tb, const Spec& C,
                       const std::string& op) {
  require(A.rank == 2 && B.rank == 2, op + ": rank-2 inputs required");
  GemmArgs g;
  g.ta = ta;
  g.tb = tb;
  g.M = ta ? A.shape[1] : A.shape[0];
  g.K = ta ? A.shape[0] : A.shape[1];
  int64_t kb = tb ? B.shape[1] : B.shape[0];
  g.N = tb ? B.shape[0] : B.shape[1];
  if (g.K != kb)
    fail(TCB_ERR_TYPE, op + ": inner dimensions disagree");
  require(A.dtype == B.dtype, op + ": dtype mismatch without explicit cast");
  require(is_float(A.dtype), op + ": float operands only");
  require(C.rank == 2 && C.shape[0] == g.M && C.shape[1] == g.N, op + ": output shape mismatch");
  g.a.ld = A.shape[1];
  g.b.ld = B.shape[1];
  g.a.dtype = A.dtype;
  g.b.dtype = B.dtype;
  g.ldc = g.N;
  g.c_dtype = C.dtype;
  return g;
}

// optional tile override: attrs tc_bn / tc_cg (parity tests cover every variant)
static void tile_attrs(GemmArgs& g, const Plan& p) {
  g.force_bn = int(p.attrs.i("tc_bn", 0));
  g.force_cg = int(p.attrs.i("tc_cg", 0));
  g.trace = reinterpret_cast<void*>(p.attrs.i("tc_trace", 0));  // tooling only
  g.no_tma_epi = int(p.attrs.i("tc_notma", 0));
  g.generic_epi = int(p.attrs.i("tc_generic_epi", 0));
}

static void b_matmul(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  GemmArgs g = gemm2d(p.in[0], p.in[1], 0, 0, p.out[0], "matmul");
  require(p.out[0].dtype == p.in[0].dtype, "matmul: output dtype must equal input dtype");
  const bool exact = want_exact(p);
  auto keep = std::make_shared<GemmWs>();
  gemm_prepare(g, exact, *keep);
  p.run = [g, exact, keep](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) mutable {
    g.a.ptr = in[0].ptr;
    g.b.ptr = in[1].ptr;
    g.c = out[0].ptr;
    launch_gemm(g, exact, s);
  };
}
TCB_REGISTER("matmul", b_matmul);

static void b_matmul_t(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  GemmArgs g = gemm2d(p.in[0], p.in[1], int(p.attrs.i("ta", 0)), int(p.attrs.i("tb", 0)), p.out[0],
                      "matmul_t");
  tile_attrs(g, p);
  g.alpha = float(p.attrs.f("alpha", 1.0));
  const bool exact = want_exact(p);
  auto keep = std::make_shared<GemmWs>();
  gemm_prepare(g, exact, *keep);
  p.run = [g, exact, keep](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) mutable {
    g.a.ptr = in[0].ptr;
    g.b.ptr = in[1].ptr;
    g.c = out[0].ptr;
    launch_gemm(g, exact, s);
  };
}
TCB_REGISTER("matmul_t", b_matmul_t);

static void b_linear(Plan& p) {
  check_arity(p, 3, 3, 1, 2);
  GemmArgs g = gemm2d(p.in[0], p.in[1], 0, int(p.attrs.i("tw", 0)), p.out[0], "linear");
  tile_attrs(g, p);
  require(p.in[2].numel() == g.N, "linear: bias must have N elements");
  g.bias_dtype = p.in[2].dtype;
  g.act = parse_act(p.attrs.s("act", "none"));
  if (p.out.size() > 1) require(same_shape(p.out[1], p.out[0]) && p.out[1].dtype == p.out[0].dtype,
                                "linear: pre-activation output must match y");
  const bool exact = want_exact(p);
  const bool save = p.out.size() > 1;
  // save=grad: the second output is act'(u) (the backward then multiplies by it)
  const std::string what = p.attrs.s("save", "preact");
  require(what == "preact" || what == "grad", "linear: save must be preact or grad");
  g.save_grad = what == "grad" ? 1 : 0;
  if (g.save_grad) require(save && g.act != ACT_NONE, "linear: save=grad needs an activation and two outputs");
  auto keep = std::make_shared<GemmWs>();
  gemm_prepare(g, exact, *keep);
  p.run = [g, exact, save, keep](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) mutable {
    g.a.ptr = in[0].ptr;
    g.b.ptr = in[1].ptr;
    g.bias = in[2].ptr;
    g.c = out[0].ptr;
    g.aux_out = save ? out[1].ptr : nullptr;
    launch_gemm(g, exact, s);
  };
}
TCB_REGISTER("linear", b_linear);

static void b_matmul_dact(Plan& p) {
  check_arity(p, 3, 3, 1, 1);
  GemmArgs g = gemm2d(p.in[0], p.in[1], int(p.attrs.i("ta", 0)), int(p.attrs.i("tb", 0)), p.out[0],
                      "matmul_dact");
  tile_attrs(g, p);
  g.dact = parse_act(p.attrs.s("act", "none"));
  require(same_shape(p.in[2], p.out[0]), "matmul_dact: aux must have the output's shape");
  g.aux_dtype = p.in[2].dtype;
  const bool exact = want_exact(p);
  auto keep = std::make_shared<GemmWs>();
  gemm_prepare(g, exact, *keep);
  p.run = [g, exact, keep](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) mutable {
    g.a.ptr = in[0].ptr;
    g.b.ptr = in[1].ptr;
    g.aux = in[2].ptr;
    g.c = out[0].ptr;
    launch_gemm(g, exact, s);
  };
}
TCB_REGISTER("matmul_dact", b_matmul_dact);

// matmul_pair(a0, b0 [, aux0], a1, b1): two independent GEMMs, one persistent
// launch (launch_gemm_tc_pair); any other dtype runs them back to back
static void b_matmul_pair(Plan& p) {
  const int n0 = int(p.attrs.i("n0", 2));
  require(n0 == 2 || n0 == 3, "matmul_pair: n0 must be 2 or 3");
  check_arity(p, n0 + 2, n0 + 2, 2, 2);
  GemmArgs g0 = gemm2d(p.in[0], p.in[1], int(p.attrs.i("ta0", 0)), int(p.attrs.i("tb0", 0)), p.out[0], "matmul_pair");
  GemmArgs g1 = gemm2d(p.in[n0], p.in[n0 + 1], int(p.attrs.i("ta1", 0)), int(p.attrs.i("tb1", 0)), p.out[1],
                       "matmul_pair");
  g0.alpha = float(p.attrs.f("alpha0", 1.0));
  g1.alpha = float(p.attrs.f("alpha1", 1.0));
  if (n0 == 3) {
    g0.dact = parse_act(p.attrs.s("act0", "none"));
    require(same_shape(p.in[2], p.out[0]), "matmul_pair: aux0 must have output 0's shape");
    g0.aux_dtype = p.in[2].dtype;
  }
  g0.force_bn = g1.force_bn = int(p.attrs.i("tc_bn", 0));
  g0.force_cg = g1.force_cg = int(p.attrs.i("tc_cg", 0));
  g0.trace = g1.trace = reinterpret_cast<void*>(p.attrs.i("tc_trace", 0));  // tooling only
  g0.generic_epi = g1.generic_epi = int(p.attrs.i("tc_generic_epi", 0));
  const bool exact = want_exact(p) || p.in[n0].dtype != TCB_BF16;
  p.nkernels = exact ? 2 : 1;
  std::shared_ptr<Scratch> sched;  // read-only schedule table
  size_t wsbuf = 0;                // K-slice partials (workspace)
  int ws_idx = -1, ws_s = 1;
  if (!exact && !p.attrs.i("static_rr", 0)) {
    // a weight gradient with few long tiles is cut along K into slices
    // (partials in a plan-owned workspace, reduced in slice order afterwards)
    const int forced = int(p.attrs.i("wsplit", 0));  // tests / tuning (1 disables)
    for (int i = 0; i < 2 && ws_s == 1; ++i) {
      const GemmArgs& g = i ? g1 : g0;
      const int sp = forced ? forced : gemm_pair_wsplit(g0, g1, i);
      if (sp > 1 && gemm_wsplit_ok(g, sp)) {
        ws_idx = i;
        ws_s = sp;
      }
    }
    if (ws_s > 1) {
      GemmArgs& g = ws_idx ? g1 : g0;
      g.wsplit = ws_s;
      wsbuf = p.ws_take(size_t(ws_s) * size_t(g.M) * size_t(g.N) * sizeof(float));
      p.nkernels = 2;
    }
    int rounds = 0;
    std::vector<int> table = gemm_pair_schedule(g0, g1, &rounds);
    sched = std::make_shared<Scratch>(table.size() * sizeof(int));
    TCB_CUDA(cudaMemcpy(sched->p, table.data(), table.size() * sizeof(int), cudaMemcpyHostToDevice));
    g0.sched = static_cast<const int*>(sched->p);
    g0.sched_rounds = rounds;
  }
  p.run = [g0, g1, exact, n0, sched, wsbuf, ws_idx, ws_s](const tcb_tensor* in, tcb_tensor* out,
                                                          cudaStream_t s) mutable {
    g0.a.ptr = in[0].ptr;
    g0.b.ptr = in[1].ptr;
    if (n0 == 3) g0.aux = in[2].ptr;
    g0.c = out[0].ptr;
    g1.a.ptr = in[n0].ptr;
    g1.b.ptr = in[n0 + 1].ptr;
    g1.c = out[1].ptr;
    if (!exact && gemm_tc_supported(g0, nullptr) && gemm_tc_supported(g1, nullptr)) {
      if (ws_s > 1) (ws_idx ? g1 : g0).c = ws_at(wsbuf);
      launch_gemm_tc_pair(g0, g1, s);
      if (ws_s > 1) {
        const GemmArgs& g = ws_idx ? g1 : g0;
        launch_wsplit_reduce(static_cast<const float*>(ws_at(wsbuf)), static_cast<float*>(out[ws_idx].ptr), g.M * g.N,
                             ws_s, s);
      }
    } else {
      g0.wsplit = g1.wsplit = 1;
      launch_gemm(g0, exact, s);
      launch_gemm(g1, exact, s);
    }
  };
}
TCB_REGISTER("matmul_pair", b_matmul_pair);

static void b_batch_matmul(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  const Spec &A = p.in[0], &B = p.in[1], &C = p.out[0];
  require(A.rank == 3 && B.rank == 3 && C.rank == 3, "batch_matmul: rank-3 inputs required");
  require(A.shape[0] == B.shape[0] && C.shape[0] == A.shape[0], "batch_matmul: batch mismatch");
  GemmArgs g;
  g.ta = int(p.attrs.i("ta", 0));
  g.tb = int(p.attrs.i("tb", 0));
  g.M = g.ta ? A.shape[2] : A.shape[1];
  g.K = g.ta ? A.shape[1] : A.shape[2];
  g.N = g.tb ? B.shape[1] : B.shape[2];
  require((g.tb ? B.shape[2] : B.shape[1]) == g.K, "batch_matmul: inner dimensions disagree");
  require(C.shape[1] == g.M && C.shape[2] == g.N, "batch_matmul: output shape mismatch");
  require(A.dtype == B.dtype, "batch_matmul: dtype mismatch");
  g.Z = A.shape[0];
  g.Z2 = 1;
  g.a.ld = A.shape[2];
  g.b.ld = B.shape[2];
  g.a.s1 = A.shape[1] * A.shape[2];  // z1 = z when Z2 == 1
  g.b.s1 = B.shape[1] * B.shape[2];
  g.c_s1 = g.M * g.N;
  g.a.dtype = A.dtype;
  g.b.dtype = B.dtype;
  g.ldc = g.N;
  g.c_dtype = C.dtype;
  g.alpha = float(p.attrs.f("alpha", 1.0));
  tile_attrs(g, p);
  const bool exact = want_exact(p);
  auto keep = std::make_shared<GemmWs>();
  gemm_prepare(g, exact, *keep);
  p.run = [g, exact, keep](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) mutable {
    g.a.ptr = in[0].ptr;
    g.b.ptr = in[1].ptr;
    g.c = out[0].ptr;
    launch_gemm(g, exact, s);
  };
}
TCB_REGISTER("batch_matmul", b_batch_matmul);

}  // namespace tcb
