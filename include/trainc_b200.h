/* trainc_b200.h -- C ABI of libtrainc_b200.so, the C++ host runtime that runs
 * the reference's compiled training step on the b200 dialect.
 *
 * The library is built against the reference's own IR / op registry /
 * KernelCache headers (/root/reference/proj/include/trainc) and links
 * libtcb200.so (include/tcb200.h).  Each entry point replaces a piece of the
 * reference's driver surface:
 *
 *   tb_session_create   <- `trainc compile` + vm::compile (A.1-A.7
 *                          of SURVEY.md §3): build -> autodiff -> fusion ->
 *                          [schedule] -> [remat under budget] -> dispatch to b200
 *   tb_session_step     <- vm::run of the all-in-one step function
 *   tb_graph_info/text  <- `trainc inspect` (IR, bytecode, memory curve) on CPU
 *   tb_text_reprint     <- parse_text / print_text (text.hpp:156-160, :620) with
 *                          bf16 / i32 parameter tokens (host/text_ext.hpp)
 *   tb_tnsr_*           <- save_tensor / load_tensor (tensor.hpp:76-139), with the
 *                          bf16 (2) and i32 (3) extension codes
 *   tb_session_save_param / load_param
 *                       <- the TNSR parameter dumps of `trainc train` (checkpoint /
 *                          resume of params, bf16 copy, Adam m/v, step)
 *   tb_autocast_info    <- the autocast + place_casts passes
 *   tb_cache_stats/clear <- KernelCache::compiles/hits/size/clear
 *                          (backends.hpp:356-368)
 *
 * Conventions: int returns are 0 on success, nonzero with tb_last_error() set
 * (the reference exception's what() string).  Session handles are opaque.
 */
#ifndef TRAINC_B200_H_
#define TRAINC_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* tb_last_error(void);

/* CPU-only graph inspection (no device): cfg is "kind=bert;L=12;H=768;..." */
int tb_graph_info(const char* cfg, int64_t* out, int n);
const char* tb_graph_text(const char* cfg, const char* what); /* "ir" | "text" | "mem" */
const char* tb_text_reprint(const char* text); /* parse (text.hpp + bf16/i32) -> print */

/* device session: compiled step + static arena + state on `device` */
void* tb_session_create(const char* cfg, int device);
void tb_session_destroy(void* h);
int tb_session_info(void* h, int64_t* out, int n);
int tb_session_init_params(void* h);
int tb_synthetic_batch(int64_t T, int64_t V, int64_t seed, int32_t* ids, int32_t* labels, int causal_lm);
int tb_session_set_batch(void* h, const int32_t* ids, const int32_t* labels);
int32_t* tb_session_ids_buffer(void* h);
int32_t* tb_session_labels_buffer(void* h);
int tb_session_step(void* h, int use_graph);
int tb_session_fetch_loss(void* h);
float tb_session_loss_value(void* h);
int tb_session_sync(void* h);
void* tb_session_stream(void* h);
int tb_session_param(void* h, const char* name, void** ptr, int64_t* bytes);
const char* tb_session_segments(void* h);
const char* tb_session_text(void* h, const char* what);
int tb_session_set_comm(void* h, void* comm);
/* vm.profile: per-instruction median device time over `repeats` eager steps
 * (CSV idx,op,let,median_us,bytes_in,bytes_out,kernels); NULL on error */
const char* tb_session_profile(void* h, int repeats);
/* ... each launch instruction run `inner` times back to back between its
 * events (the per-launch mean); advances the training state `inner` updates */
const char* tb_session_profile_inner(void* h, int repeats, int inner);

/* AutoCast pass census on the all-f32 step (CPU only; host/autocast.hpp) */
int tb_autocast_info(const char* cfg, const char* policy, const char* placement, int64_t* out, int n);

/* memsched on a text-IR function (CPU only; host/memsched.hpp):
 * what = "liveness" | "curve" | "schedule" | "remat" (under budget bytes);
 * transient_inputs: inputs die at their last use (SPEC.md example accounting).
 * Returns NULL on error (tb_last_error). */
const char* tb_memsched_text(const char* text, const char* what, int64_t budget, int transient_inputs);

/* backends::derive_priorities over "dialect op shape_class median_us" lines
 * (e.g. from tb_session_profile); returns "dialect.op priority" lines */
const char* tb_derive_priorities(const char* samples);

/* KernelCache */
int tb_cache_clear(void); /* only with no session alive */
int tb_cache_stats(int64_t* out3);

/* TNSR files: "TNSR", u8 code, u8 rank, u64 dims, raw LE data.
 * code 0 f32, 1 f16 (reference), 2 bf16, 3 i32 (extension). */
int tb_tnsr_save(const char* path, const void* data, int code, int rank, const int64_t* shape);
int tb_tnsr_header(const char* path, int* code, int* rank, int64_t* shape, int cap);
int tb_tnsr_load(const char* path, void* data, int64_t bytes);
int tb_session_save_param(void* h, const char* name, const char* path);
int tb_session_load_param(void* h, const char* name, const char* path);

#ifdef __cplusplus
}
#endif

#endif /* TRAINC_B200_H_ */
