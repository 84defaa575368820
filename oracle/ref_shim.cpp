// ref_shim.cpp -- C entry points over the UNMODIFIED reference kernels
// (TEST INFRASTRUCTURE).  Compiled by oracle/Makefile directly against the
// headers under /root/reference/proj/include into oracle/_ref/libtrainc_ref.so;
// no reference source is copied into this repository.
//
// ref_exec() runs trainc::backends::exec_base (backends.hpp:162-275), the `ref`
// dialect; ref_exec_opt() runs the opt dialect kernels matmul_blocked
// (backends.hpp:280-304) and matmul_add_act (backends.hpp:311-324).  Both take
// the same tensor/attr structs as oracle.h so tests can compare the CPU
// restatement (oracle.c) with the reference bit for bit.
#include <cstring>
#include <string>

#include "trainc/backends.hpp"
#include "../oracle/oracle.h"

using namespace trainc;

static thread_local std::string g_err;

static TensorType to_type(const orc_tensor& t) {
  TensorType ty;
  ty.dtype = t.dtype == ORC_F16 ? DType::F16 : DType::F32;
  for (int i = 0; i < t.rank; ++i) ty.shape.push_back(t.shape[i]);
  return ty;
}

static Tensor to_tensor(const orc_tensor& t) {
  TensorType ty = to_type(t);
  Tensor x(ty);
  const float* p = static_cast<const float*>(t.ptr);
  for (size_t i = 0; i < x.data.size(); ++i) x.data[i] = p[i];
  return x;
}

static ir::AttrMap to_attrs(const orc_attr* a, int na) {
  ir::AttrMap m;
  for (int i = 0; i < na; ++i) {
    if (a[i].kind == 0) m[a[i].key] = std::int64_t(a[i].i);
    else if (a[i].kind == 1) m[a[i].key] = a[i].d;
    else m[a[i].key] = std::string(a[i].s ? a[i].s : "");
  }
  return m;
}

static void copy_out(const Tensor& t, orc_tensor& o) {
  std::memcpy(o.ptr, t.data.data(), t.data.size() * sizeof(float));
}

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_exec(const char* op, const orc_tensor* in, int nin, orc_tensor* out, int nout,
             const orc_attr* attrs, int na) {
  try {
    TensorList xs;
    for (int i = 0; i < nin; ++i) xs.push_back(to_tensor(in[i]));
    Type out_ty;
    if (nout == 1 && std::string(op) != "reduce_scatter_batched" &&
        std::string(op) != "all_gather_batched") {
      out_ty = to_type(out[0]);
    } else {
      TupleType tt;
      for (int i = 0; i < nout; ++i) tt.fields.push_back(to_type(out[i]));
      out_ty = tt;
    }
    TensorList ys = backends::exec_base(op, to_attrs(attrs, na), xs, out_ty);
    for (int i = 0; i < nout && i < (int)ys.size(); ++i) copy_out(ys[i], out[i]);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// act: 0 none (plain matmul_blocked), 1 relu, 2 tanh; bias may be NULL for act 0.
int ref_exec_opt(const orc_tensor* a, const orc_tensor* b, const orc_tensor* bias, int act,
                 orc_tensor* out) {
  try {
    Tensor A = to_tensor(*a), B = to_tensor(*b);
    TensorType ot = to_type(*out);
    Tensor C;
    if (!bias) {
      C = backends::matmul_blocked(A, B, ot);
    } else {
      backends::Epilogue e = act == 1 ? backends::Epilogue::Relu
                             : act == 2 ? backends::Epilogue::Tanh
                                        : backends::Epilogue::None;
      C = backends::matmul_add_act(A, B, to_tensor(*bias), ot, e);
    }
    copy_out(C, *out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Reference f16 conversion (fp16.hpp:14-76), for the exhaustive 65,536-pattern test.
uint16_t ref_float_to_half_bits(float f) { return float_to_half_bits(f); }
float ref_half_bits_to_float(uint16_t h) { return half_bits_to_float(h); }

// trainc::Rng (tensor.hpp:145-176) draws, for pinning the oracle's mt19937.
void ref_rng_fill_uniform(uint64_t seed, float* out, int64_t n, float lo, float hi) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}
void ref_rng_fill_below(uint64_t seed, int32_t* out, int64_t n, uint32_t bound) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<int32_t>(r.below(bound));
}

// Reference type relations (opreg.hpp:278-497): output shape of `op` for the
// given input types, written as rank + dims into shape_out (one tensor result)
// or -1 for tuples; used to pin the host-side type relations.
int ref_infer(const char* op, const orc_tensor* in, int nin, const orc_attr* attrs, int na,
              int64_t* shape_out, int* rank_out, int* dtype_out) {
  try {
    std::vector<Type> ts;
    for (int i = 0; i < nin; ++i) ts.push_back(to_type(in[i]));
    Type t = opreg::registry().type_rel_of(op)(ts, to_attrs(attrs, na));
    if (!t.is_tensor()) {
      *rank_out = -1;
      return 0;
    }
    *rank_out = t.tensor().rank();
    *dtype_out = t.tensor().dtype == DType::F32 ? 0 : 1;
    for (int i = 0; i < *rank_out; ++i) shape_out[i] = t.tensor().shape[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// trainc::save_tensor / load_tensor (tensor.hpp:80-133) on float host data:
// f16 tensors are passed as floats and rounded by the reference on save.
int ref_tnsr_save(const char* path, const float* data, int code, int rank, const int64_t* shape) {
  try {
    TensorType ty;
    ty.dtype = code == 1 ? DType::F16 : DType::F32;
    for (int i = 0; i < rank; ++i) ty.shape.push_back(shape[i]);
    Tensor t(ty);
    for (size_t i = 0; i < t.data.size(); ++i) t.data[i] = data[i];
    save_tensor(t, std::string(path));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// out must hold cap floats; *code/*rank/shape[0..rank) describe the file
int ref_tnsr_load(const char* path, float* out, int64_t cap, int* code, int* rank, int64_t* shape) {
  try {
    Tensor t = load_tensor(std::string(path));
    *code = t.ty.dtype == DType::F32 ? 0 : 1;
    *rank = t.ty.rank();
    for (int i = 0; i < *rank && i < 8; ++i) shape[i] = t.ty.shape[size_t(i)];
    if (int64_t(t.data.size()) > cap) throw Error("ref_tnsr_load: buffer too small");
    std::memcpy(out, t.data.data(), t.data.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
