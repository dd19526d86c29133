/* dlvm.h -- C ABI of the B200-native DLVM hot path.
 *
 * What it computes: a straight-line DLVM IR function (§3.1.1
 * L200-218, instruction set Table 1) and the gradient function the
 * paper's AD pass generates from a gradient declaration (§3.1.3,
 * Fig. 3): "The canonicalization process first copies basic blocks
 * and instructions from the original function to the new function body, and
 * then applies adjoint code generation" (L296).  A handle is the
 * shape-specialised, "reified" callable of NNKit's JIT (§3.4):
 * parse -> verify -> differentiate -> dead-code-eliminate -> plan fused
 * sm_100a launches, once, at create time.
 *
 * Conventions (all entry points):
 *  - No C++ exception crosses this boundary.  Every call returns a
 *    dlvm_status; on failure dlvm_last_error() holds a thread-local message
 *    "line:col: error: ..." (line/col 0 when not tied to the text).
 *  - Tensors are dense, row-major, with `data` 16-byte aligned.  All device
 *    memory (inputs, outputs, seed, workspace) is CALLER-OWNED (e.g. torch)
 *    and must stay alive until the work queued on `cuda_stream` completes.
 *    The library allocates no device memory and never synchronises the host
 *    in dlvm_fn_run / dlvm_grad_run, so both are CUDA-graph capturable.
 *  - A handle is not re-entrant (the workspace is shared): one handle per
 *    stream.  Handles are immutable after create and may be destroyed from
 *    any thread once their work has completed.
 *  - Shapes are static (NNKit "shape-specialized DLVM IR"): tensors
 *    passed to run must match the signature exactly (DLVM_ERR_USAGE).
 */
#ifndef DLVM_H_
#define DLVM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; 0-4 mirror the exit codes of SPEC.md L557-559. */
typedef enum {
  DLVM_OK = 0,
  DLVM_ERR_VERIFY = 1,      /* type/shape/gradient-declaration error (create) */
  DLVM_ERR_PARSE = 2,       /* malformed IR text (create) */
  DLVM_ERR_USAGE = 3,       /* bad arguments: arity, shape, dtype, NULL handle */
  DLVM_ERR_RUNTIME = 4,     /* internal planner/executor failure */
  DLVM_ERR_CUDA = 5,        /* a CUDA launch or driver call failed */
  DLVM_ERR_UNSUPPORTED = 6  /* valid IR outside what the GPU path executes */
} dlvm_status;

/* Element types of caller tensors.  IR `bool` is stored one byte per element
 * (0/1).  DLVM_BF16 is a storage type, not an IR type (reading A15 of
 * SURVEY.md §8(c)): an f32 argument may be passed as bf16 -- its values are
 * then exactly the f32 widening of the bf16 elements (e.g. one-hot targets,
 * or operands the bf16 dot policy rounds anyway) -- under DLVM_DOT_BF16, or
 * under DLVM_DOT_F32 if it feeds no `dot`.  An f32 argument that feeds no
 * `dot` may also be passed as DLVM_BOOL bytes: its values are then 1.0
 * where the byte is nonzero, else 0.0 (exact for 0/1 data such as one-hot
 * targets or masks).  An f32 output may be requested as bf16 (stored with
 * round-to-nearest-even). */
typedef enum { DLVM_BOOL = 0, DLVM_F32 = 1, DLVM_F64 = 2, DLVM_BF16 = 3, DLVM_F32_ADD = 4 } dlvm_dtype;
/* DLVM_F32_ADD (outputs only): an f32 output the kernels ACCUMULATE into
 * with red.global.add instead of storing -- the fused gradient reduction of
 * the data-parallel path: `data` may be a peer
 * GPU's memory reachable over NVLink (P2P / symmetric memory), so every
 * rank adds its partial gradient straight into the owner's buffer from the
 * GEMM epilogue (or the element-wise step that finalises it).  The caller
 * zeroes the buffer first and orders every contributor's run before reading
 * it.  Floating-point addition order across concurrent contributors is not
 * fixed (two contributors into a zeroed buffer are order-independent).
 * Rejected (DLVM_ERR_USAGE) for outputs a later launch reads back. */

#define DLVM_MAX_RANK 8
typedef struct {
  void* data;                    /* device pointer (caller-owned) */
  int32_t dtype;                 /* dlvm_dtype */
  int32_t rank;                  /* 0..DLVM_MAX_RANK; 0 = scalar */
  int64_t shape[DLVM_MAX_RANK];
} dlvm_tensor;

/* dot precision policy (reading A15) */
#define DLVM_DOT_F32 0   /* exact fp32 operands, FFMA accumulation */
#define DLVM_DOT_BF16 1  /* bf16 operands (RNE), fp32 accumulation in TMEM (tcgen05) */

/* option flags */
#define DLVM_PLAN_ONLY 0x1u      /* parse/verify/differentiate/plan only; no device calls */
#define DLVM_NO_FUSION 0x2u      /* one launch group per instruction (testing) */
#define DLVM_NO_SPECIALIZE 0x4u  /* always use the generic element-wise program interpreter */
#define DLVM_NO_OPT 0x8u         /* skip the create-time IR optimiser (algebra simplification, CSE,
                                    matrix-chain reordering; §3.1.2) */
#define DLVM_NO_JIT 0x10u        /* no create-time NVRTC specialisation of element-wise programs that
                                    are not in the ahead-of-time registry (they are interpreted) */

typedef struct {
  int32_t dot_precision; /* DLVM_DOT_F32 | DLVM_DOT_BF16 */
  int32_t device;        /* -1: launch on the caller's current device (the default);
                            >= 0: create loads its kernels into, and run/grad_run launch on,
                            that device (made current for the call, then restored).  The
                            tensors and stream passed to run must live on that device. */
  uint32_t flags;        /* DLVM_PLAN_ONLY | DLVM_NO_FUSION | DLVM_NO_SPECIALIZE | DLVM_NO_OPT | DLVM_NO_JIT */
} dlvm_options;

typedef struct dlvm_fn_s* dlvm_fn;

/* Which function of a handle. */
#define DLVM_PRIMAL 0
#define DLVM_GRADIENT 1

/* Defined by: the module/function/gradient-declaration structure of Fig. 3
 * (P:L246-272), the canonicalisation of a gradient declaration into a
 * function -- "first copies basic blocks and instructions from the original
 * function to the new function body, and then applies adjoint code
 * generation" (§3.1.3) -- and NNKit's shape-specialised lowering and
 * "function reification" (§3.4): a handle is that reified,
 * shape-specialised callable.
 * Parse `module_text` (len bytes, need not be NUL-terminated), verify the
 * whole module, and build a handle for function `fn_name` and, if
 * `grad_name` is non-NULL, the gradient declaration of that name (which must
 * be a `[gradient @fn_name ...]` declaration); with grad_name NULL the unique
 * gradient declaration of fn_name is used if there is exactly one.
 * Errors: DLVM_ERR_PARSE, DLVM_ERR_VERIFY (incl. non-differentiable),
 * DLVM_ERR_UNSUPPORTED (e.g. f64/integer tensors on the GPU path),
 * DLVM_ERR_USAGE (NULL pointers, unknown function names, device < -1),
 * DLVM_ERR_CUDA (cudaSetDevice for opts->device failed).  `opts` may be NULL
 * (defaults: DLVM_DOT_F32, device -1 = current, no flags).  Ownership: *out
 * is a host-side object owned by the caller until dlvm_fn_destroy; *out is
 * NULL on failure. */
dlvm_status dlvm_fn_create(const char* module_text, size_t len, const char* fn_name,
                           const char* grad_name, const dlvm_options* opts, dlvm_fn* out);

/* Defined by: the function types of Fig. 3 -- `@foo: (<1x784>, <784x10>,
 * <1x10>) -> <1x10>`, `@foo_grad` and the seedable
 * `@foo_grad_3` with its seed appended and results (dW, db, kept)
 * -- and Table 1's type rules.
 * Inferred signature of the primal (which=0) or gradient (which=1) function.
 * On entry *n_in / *n_out hold the capacity of in_types / out_types (either
 * array may be NULL with capacity 0 to query counts); on exit they hold the
 * counts.  Returned tensors have data=NULL and dtype DLVM_F32/DLVM_F64/
 * DLVM_BOOL as typed in the IR.  Gradient outputs are ordered: gradients in
 * `wrt` order, then `keeping` outputs (Fig. 3, Fig. 4). */
dlvm_status dlvm_fn_signature(dlvm_fn fn, int which, int* n_in, dlvm_tensor* in_types, int* n_out,
                              dlvm_tensor* out_types);

/* Text of the typed primal (which=0), the generated gradient function after
 * dead-code elimination (which=1) in the .dl syntax of Fig. 3, the launch
 * plan of the primal (2) / gradient (3), the element-wise program
 * signatures of the primal (4) / gradient (5) launches (one per line, the
 * keys of the compile-time specialisations), the optimised primal (6) /
 * gradient (7) that the plans execute (identical to 0/1 with DLVM_NO_OPT),
 * (8) the kernels specialised at create time by NVRTC (one line each:
 * plan, step, status, instantiation), or the detailed plan of the primal (9)
 * / gradient (10): buffers, then every step's iteration space, launch shape,
 * program signature and operand refs (buffer, offset, strides, chunks), or
 * the two-stream schedule of the primal (11) / gradient (12): per step the
 * stream (the caller's, or the handle's auxiliary stream running an
 * independent GEMM beside the previous one) and its cross-stream waits.
 * Writes at most `cap` bytes
 * including the NUL; *needed receives the full size including the NUL. */
dlvm_status dlvm_fn_print(dlvm_fn fn, int which, char* buf, size_t cap, size_t* needed);

/* Device workspace bytes dlvm_fn_run (which=0) / dlvm_grad_run (which=1)
 * need; the caller passes a buffer at least this large (256-byte aligned).
 * The workspace holds intermediates of one run: concurrent runs (e.g. on
 * different streams) need separate workspaces.  Errors: DLVM_ERR_USAGE
 * (NULL handle/pointer, which not 0/1, which=1 without a gradient). */
dlvm_status dlvm_fn_workspace_bytes(dlvm_fn fn, int which, size_t* bytes);

/* Number of kernel launches one run (which=0) / grad run (which=1) issues
 * with every output bound as f32.  Binding an output that a single-partial
 * reduction produces as bf16 adds one small finalize launch for it (not
 * covered by dlvm_fn_launch_events). */
dlvm_status dlvm_fn_num_launches(dlvm_fn fn, int which, int* launches);

/* Defined by: the instruction semantics of §3.1.1 and Table 1
 * (P:L164-189), evaluated in program order ("straight-line" function).
 * Execute the primal function on `cuda_stream` (a cudaStream_t; NULL = the
 * legacy default stream).  in[n_in] / out[n_out] follow the signature; the
 * caller owns every buffer and keeps it alive until the stream's work is
 * done.  Errors (returned before anything is queued): DLVM_ERR_USAGE for
 * arity, shape, dtype, alignment or NULL-workspace mismatches;
 * DLVM_ERR_UNSUPPORTED if the function could not be planned; DLVM_ERR_CUDA
 * if a launch fails (earlier launches of the call may already be queued).
 * Device faults surface asynchronously at the caller's next sync. */
dlvm_status dlvm_fn_run(dlvm_fn fn, const dlvm_tensor* in, int n_in, dlvm_tensor* out, int n_out,
                        void* workspace, void* cuda_stream);

/* Defined by: the gradient declaration (§3.1.3): a function
 * that "takes original inputs and produces a tuple of partial derivatives
 * with respect to the inputs", i.e. the vector-Jacobian product
 * seed^T J_f restricted to `wrt` (reading A6), configurable by
 * `wrt`, `keeping`, `from` and `seedable`, with unused
 * operations removed by dead-code elimination.
 * Execute the gradient function.  `in` holds the primal arguments; `seed`
 * is non-NULL iff the declaration is `seedable` (it is the last parameter of
 * the gradient function).  out[n_out]: gradients in `wrt` order, then kept
 * outputs.  If `grad_ready_events` is non-NULL it points to n_grads
 * cudaEvent_t (n_grads = number of `wrt` gradients), each recorded on
 * `cuda_stream` as soon as that gradient is final -- a communication stream
 * can wait on them to overlap a gradient all-reduce with the rest of the
 * adjoint (data-parallel path).  Ownership and errors as
 * for dlvm_fn_run; events are caller-owned and must be real (created)
 * cudaEvent_t handles. */
dlvm_status dlvm_grad_run(dlvm_fn fn, const dlvm_tensor* in, int n_in, const dlvm_tensor* seed,
                          dlvm_tensor* out, int n_out, void* workspace, void* cuda_stream,
                          void* const* grad_ready_events);

/* Profiling hook.  With n_events == dlvm_fn_num_launches(fn, which) + 1,
 * every later run of `which` records events[i] (cudaEvent_t) on its stream
 * right before launch i and events[n_events-1] after the last launch, so a
 * caller can time each kernel with cudaEventElapsedTime on the launching
 * stream.  events == NULL (or n_events == 0) disables it.  The handle keeps
 * the pointer array; the caller keeps it and the events alive while set. */
dlvm_status dlvm_fn_launch_events(dlvm_fn fn, int which, void* const* events, int n_events);

/* Short description ("gemm tcgen05 bf16 %z1 M=... N=... K=...", "ew [...]")
 * of launch i of `which`, and its algorithmic work: flops (2*M*N*K for a
 * GEMM, 0 otherwise) and the bytes it must move at minimum (every input
 * element read once, every output element written once). */
dlvm_status dlvm_fn_launch_info(dlvm_fn fn, int which, int i, char* buf, size_t cap, double* flops,
                                double* bytes);

/* Defined by: SPEC.md's diagnostics format "line:col: severity: message"
 * (S:L284).  Thread-local text of the last error on this thread ("" if
 * none); the pointer stays valid until the next failing call on this
 * thread.  Never NULL. */
const char* dlvm_last_error(void);

/* Release the host-side plan.  NULL is ignored.  Work already queued by the
 * handle is unaffected (its launches hold their parameters by value, and
 * create-time NVRTC kernels stay loaded in a per-process cache); any later
 * call with the handle is invalid. */
void dlvm_fn_destroy(dlvm_fn fn);

/* Library version string, e.g. "dlvm-b200 0.1 sm_100a". */
const char* dlvm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DLVM_H_ */
