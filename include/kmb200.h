/*
 * kmb200.h — C ABI of the B200 μ-mode hot path (libkmb200.so).
 *
 * The reference (`kronmode` 0.1.0, /root/reference/pkg/src/kronmode) is pure
 * Python on numpy; its hot path has no FFI of its own — every product ends in
 * `np.matmul` (tensor.py:129, tensor.py:139).  This header is the boundary a
 * host binding crosses instead: plain device pointers, sizes and a stream, no
 * torch or numpy types.  The Python mirror in `paper_2103_01691_b200/` binds it
 * with ctypes (see INTEGRATION.md for the binding a kronmode maintainer would
 * add).
 *
 * Conventions (all entry points):
 *   - Tensors are column-major (direction 1 fastest), as tensor.py:3-6.
 *   - Matrices L (m x n_mu) are row-major (C order), as numpy hands them over.
 *   - All pointers are DEVICE pointers; the library never allocates device
 *     memory (every scratch buffer is caller-supplied: km_tucker's ws0/ws1,
 *     the tcgen05 and norm workspaces, km_set_stream_workspace), never
 *     synchronises the host and launches only on `stream` (a cudaStream_t,
 *     NULL = legacy default stream).
 *   - Per-device set-up (shared-memory opt-ins, occupancy queries, SM counts)
 *     is cached per device id and thread safe; the CURRENT device must be the
 *     one the pointers and the stream belong to.
 *   - Return value 0 on success, KM_EINVAL for a rejected argument, KM_ECUDA
 *     for a CUDA launch/runtime failure; km_last_error() gives the message of
 *     the last failure on the calling thread.
 *   - Shapes and directions are validated by the host mirror first so that
 *     its exceptions match the reference's messages (tensor.py:62-66,
 *     102-111, 151-161); the C side re-checks only what would fault.
 */
#ifndef KMB200_H
#define KMB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KMB200_ABI_VERSION 3
#define KM_MAX_D 8

/* element types; complex values are interleaved (re, im) pairs */
enum km_dtype { KM_F32 = 0, KM_F64 = 1, KM_C64 = 2, KM_C128 = 3 };

enum km_status { KM_OK = 0, KM_EINVAL = 1, KM_ECUDA = 2 };

/* pointwise operators that can be fused into a product epilogue (post) or
 * applied as a standalone pass (pre) */
enum km_op_kind {
  KM_OP_NONE = 0,
  /* Gross–Pitaevskii nonlinear half-step, problems.py:542-545:
   *   psi <- psi * exp(i * coef * (1 - |psi|^2 / (w_1[i_1] * ... * w_d[i_d])))
   * with coef = 0.5 * half_tau; `weights[mu]` are device f64 vectors. */
  KM_OP_GPE_PHASE = 1,
  /* multiplication by a complex factor that depends on one direction only:
   *   psi <- psi * diag[i_{diag_dir}]     (diag: device c128 vector)
   * used for the time-dependent potential phase exp(-i x_3 ∫ sin^2). */
  KM_OP_DIAG = 2
};

typedef struct km_pointop {
  int32_t kind;                       /* enum km_op_kind */
  int32_t d;                          /* tensor order */
  int64_t dims[KM_MAX_D];             /* extents of the tensor the op sees */
  const double* weights[KM_MAX_D];    /* KM_OP_GPE_PHASE */
  double coef;                        /* KM_OP_GPE_PHASE */
  const void* diag;                   /* KM_OP_DIAG, c128 vector of dims[diag_dir] */
  int32_t diag_dir;                   /* KM_OP_DIAG, 0-based direction */
  int32_t repeat;                     /* KM_OP_GPE_PHASE: apply 1 (0 = 1) or 2 times in a row,
                                         e.g. step k's closing and step k+1's opening half-phase */
  /* KM_OP_GPE_PHASE, optional: the weight product over directions 1..d-1,
   * w_1[i_1]*...*w_{d-1}[i_{d-1}] accumulated left to right, as a column-major
   * device f64 vector of dims[0]*...*dims[d-2] entries.  With it the kernels
   * form the full product as inner[l] * w_d[i_d] (same rounding) without
   * per-element index divisions. */
  const double* inner_weights;
  /* optional, any kind (KM_OP_NONE included): the two-norm of the values the
   * product stores (after the op), accumulated in its epilogue instead of a
   * separate pass over the result (reference: tensor.norm "two",
   * tensor.py:169-198, as the GPE driver's drift, problems.py:596-599).  Every
   * warp of every output tile writes one partial sum to a fixed slot of
   * norm_ws (no atomics) and a one-warp kernel folds them in slot order into
   * *norm_result = sqrt(sum |value|^2): deterministic.  norm_ws holds
   * norm_ws_count doubles, at least km_norm_epilogue_slots().  Honoured by
   * km_mumode, km_mumode_split and as km_tucker's post. */
  double* norm_result;
  double* norm_ws;
  int64_t norm_ws_count;
} km_pointop;

/* doubles a km_pointop's norm_ws needs for a product with m rows and M fibers
 * (M = n_left * n_right) */
int64_t km_norm_epilogue_slots(int64_t m, int64_t fibers);

/* kernel selection (process-wide, bit flags): AUTO picks the warp-specialised
 * TMA kernels where the shape allows and balances their last wave with
 * stream-K; NO_TMA forces the cp.async kernel everywhere; NO_STREAMK keeps
 * whole tiles only (A/B testing and verification).  The stream-K tail needs a
 * scratch workspace bound to the launching stream (km_set_stream_workspace);
 * on a stream without one the products keep whole tiles.  Launches captured
 * into a CUDA graph keep whole tiles: the partials' publish flags are
 * per-launch epochs, which a replayed graph would repeat. */
enum km_kernel_policy {
  KM_POLICY_AUTO = 0,
  KM_POLICY_NO_TMA = 1,
  KM_POLICY_NO_STREAMK = 2,
  KM_POLICY_NO_TC_HALVES = 4,  /* complex64 K' in (512, 1024] on the chunked tcgen05 kernel */
  KM_POLICY_NO_PLANE_FUSION = 8 /* km_tucker: no fused first-two-products launch for small 3-D complex128 planes */
};
int km_set_kernel_policy(int policy);

/*
 * Stream-K scratch (partial accumulators + publish flags) of the persistent
 * complex128/f64 TMA kernel, in the spirit of cublasSetWorkspace: the caller
 * owns the device memory and binds it to a stream of the CURRENT device;
 * products launched on that stream may then split their last wave of tiles
 * over all SMs (stream-K).  km_stream_workspace_bytes gives the size for the
 * current device (~78 MB on 148 SMs).  Binding zeroes the flags with
 * cudaMemsetAsync on `stream`; workspace == NULL unbinds.  The workspace must
 * stay allocated until the work queued on the stream has completed (e.g.
 * allocate it stream-ordered on that stream).  One workspace per stream:
 * launches on one stream are serialised, so they may share it.
 * (No reference counterpart: tensor.py's np.matmul has no work partitioning.)
 */
int km_stream_workspace_bytes(size_t* bytes);
int km_set_stream_workspace(void* stream, void* workspace, size_t bytes);

/* ABI version and build info */
int km_abi_version(void);
const char* km_build_info(void);
const char* km_last_error(void);

/*
 * μ-mode product, out = u ×_μ L  (reference: tensor.mu_mode_product,
 * tensor.py:80-140).  The tensor is flattened to (n_left, n_mu, n_right)
 * exactly as tensor.py:132-134 does; n_left == 1 is the reference's μ=1 branch
 * (tensor.py:124-130).  `out` has shape (n_left, m, n_right).
 *
 * u_dtype / L_dtype must be of one precision (F32/C64 or F64/C128); the
 * result is complex if either operand is.  `post` (may be NULL) is fused into
 * the epilogue and sees the output tensor with extents post->dims.
 * u and out must not overlap.
 */
int km_mumode(const void* u, int u_dtype, const void* L, int L_dtype, void* out,
              int64_t m, int64_t n_left, int64_t n_mu, int64_t n_right,
              const km_pointop* post, void* stream);

/*
 * The trailing-direction product (n_right == 1) restricted to the output
 * fibers [fiber0, fiber0 + fibers): out[f + i*n_left] for those f only, with u
 * and out the full (n_left, n_mu) and (n_left, m) arrays.  Same arithmetic as
 * km_mumode for those elements.  The host pipeline (_pipeline.py) uses it to
 * finish the first output rows in fiber pieces, so their device-to-host copy
 * starts before the whole row block is done (no reference counterpart: the
 * reference's product is one np.matmul, tensor.py:136-139).
 */
int km_mumode_fibers(const void* u, int u_dtype, const void* L, int L_dtype, void* out, int64_t m,
                     int64_t n_left, int64_t n_mu, int64_t fiber0, int64_t fibers, void* stream);

/*
 * Configuration 4's potential flows folded into a complex128 propagator:
 * out[i][j] = exp(-i x_rows[i] c_b) * E[i][j] * exp(-i x_cols[j] c_a), E and
 * out row-major m x k (not overlapping), x_* device node vectors, c_a / c_b
 * the integrals of sin^2 over the two half steps.  The Strang step of
 * problems.tdpot_strang_step is then a plain km_tucker launch (no reference
 * counterpart: the reference has no configuration-4 driver).
 */
int km_diag_phase_fold(const void* E, void* out, int64_t m, int64_t k, const double* x_rows, const double* x_cols,
                       double c_a, double c_b, void* stream);

/* cudaMemcpy2DAsync(cudaMemcpyDefault) on `stream`: `height` rows of `width`
 * bytes; the host pipeline's strided device-to-host copies. */
int km_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
               void* stream);

/*
 * μ-mode product on blocked ("split") layouts — the fused pack/unpack of the
 * slab decomposition's all-to-all.  Same as km_mumode (n_left
 * must be > 1), except that
 *   - the input's contracted index j is stored in blocks of `in_block`:
 *     element (l, j, r) is at (j / in_block) * in_block_stride
 *                              + l + n_left*(j % in_block) + n_left*in_block*r;
 *   - the output's row index i is stored in blocks of `out_block`:
 *     element (l, i, r) is at (i / out_block) * out_block_stride
 *                              + l + n_left*(i % out_block) + n_left*out_block*r.
 * in_block == n_mu / out_block == m are the plain layouts.  in_block must be a
 * multiple of 16 and out_block a multiple of 8 when they split.  `post` (may be
 * NULL) is fused into the epilogue as in km_mumode; it needs the plain output
 * layout (out_block == m), the input may be blocked.
 * accumulate = 1 adds the product into `out` instead of overwriting it,
 * out = post(out + u ×_μ L), each element rounded as numpy's `out += p`
 * (kron.py:99-101, the Kronecker-sum matvec; and the K-split halves of the
 * slab step).  The DMMA kernels only (complex64 x complex64 included).
 */
int km_mumode_split(const void* u, int u_dtype, const void* L, int L_dtype, void* out,
                    int64_t m, int64_t n_left, int64_t n_mu, int64_t n_right,
                    int32_t in_block, int64_t in_block_stride, int32_t out_block,
                    int64_t out_block_stride, int32_t accumulate, const km_pointop* post,
                    void* stream);

/*
 * μ-mode product whose output blocks are stored straight into other ranks'
 * receive buffers (peer device pointers, e.g. NVLink-mapped symmetric
 * memory): the all-to-all of the slab decomposition fused into the product's
 * epilogue, so the exchange overlaps the math tile by tile.
 * Exactly one blocking applies:
 *   - out_block < m (n_left > 1): output rows [b*out_block, (b+1)*out_block)
 *     go to peers[b] + peer_offset, laid out as the plain
 *     (n_left, out_block, n_right) column-major block;
 *   - fiber_block > 0 (n_left == 1): fibers [b*fiber_block, (b+1)*fiber_block)
 *     go to peers[b] + peer_offset, as the (m, fiber_block) block.
 * in_block / in_block_stride as in km_mumode_split.  Offsets are in elements.
 * The caller orders the peers' writes before the reads (a device barrier).
 */
int km_mumode_peer(const void* u, int u_dtype, const void* L, int L_dtype, int64_t m,
                   int64_t n_left, int64_t n_mu, int64_t n_right, int32_t in_block,
                   int64_t in_block_stride, int32_t out_block, int64_t fiber_block,
                   void* const* peers, int32_t npeers, int64_t peer_offset, void* stream);

/*
 * complex64 x complex64 μ-mode product on the 5th-generation tensor cores
 * (tcgen05.mma kind::tf32, TMEM accumulator, 3xTF32 split for fp32-level
 * accuracy).  Same arguments as km_mumode plus a device workspace of at least
 * km_tc_workspace_bytes(m, n_mu) bytes (the factor's split planes).  The
 * contraction K' = 2*n_mu (n_left == 1) or n_mu (n_left > 1) runs as one
 * accumulation chain up to 512, as two folded chains up to 1024, and in
 * 64-k' chunks beyond (the tensor core's fp32 accumulation truncates, so a
 * chain's error grows with its length).  Shapes the kernels do not take
 * (n_left > 1 with n_left % 128 != 0 (% 64 for the chunked kernel),
 * n_mu % 4 != 0, odd m, a too-small workspace, KM_POLICY_NO_TMA) run the
 * DMMA path instead.
 */
int km_tc_workspace_bytes(int64_t m, int64_t n_mu, size_t* bytes);
int km_mumode_c64_tc(const void* u, const void* L, void* out, int64_t m, int64_t n_left,
                     int64_t n_mu, int64_t n_right, void* workspace, size_t workspace_bytes,
                     void* stream);

/*
 * Tucker operator / exact propagator step (reference: tensor.tucker,
 * tensor.py:143-166; kron.step, kron.py:110-121; the Strang composition
 * problems.py:548-565 when pre/post are phases).
 *
 *   out = post( pre(u) ×_1 mats[0] ×_2 ... ×_d mats[d-1] )
 *
 * mats[mu] == NULL skips that direction (tensor.py:164-165).  mats[mu] has
 * rows[mu] rows and dims[mu] columns.  ws0/ws1 are scratch buffers, each at
 * least the byte size of the largest intermediate (km_tucker_workspace()).
 * ws1 may be NULL: `out` then doubles as the second ping-pong buffer, which
 * needs every intermediate to fit in out (KM_EINVAL otherwise; always true
 * for square factors), so a step costs one state-sized workspace.  The
 * workspaces must not alias u, out or each other (KM_EINVAL).
 * pre is applied in a standalone pass, post is fused into the last product.
 */
int km_tucker(const void* u, int u_dtype, int d, const int64_t* dims,
              const void* const* mats, const int* mat_dtypes, const int64_t* rows,
              void* out, void* ws0, void* ws1,
              const km_pointop* pre, const km_pointop* post, void* stream);

/*
 * `steps` exact steps of a complex128 n1 x n2 x n3 state in ONE persistent
 * launch (reference: kron.step, kron.py:110-121, applied `steps` times; the
 * time loop of problems.py:597-598): the d = 3 sweeps of every step run as
 * one dataflow of 32 x 32 tiles whose dependencies on the previous sweep are
 * tracked by counters, so the sweeps overlap instead of paying a launch,
 * a pipeline fill and a partial last wave each (small, L2-resident states).
 * E1..E3 are the row-major n_mu x n_mu complex128 propagators; `state` is
 * updated in place.  Extents must be multiples of 32 in [32, 96]
 * (KM_EINVAL otherwise; the caller then steps with km_tucker).  The
 * workspace (two state copies + counters) is km_steps_small_workspace_bytes.
 * Not capturable into a CUDA graph (cooperative launch).
 */
int km_steps_small_workspace_bytes(int64_t n1, int64_t n2, int64_t n3, int64_t steps, size_t* bytes);
int km_steps_small(void* state, const void* E1, const void* E2, const void* E3, int64_t n1, int64_t n2,
                   int64_t n3, int64_t steps, void* workspace, size_t workspace_bytes, void* stream);

/*
 * `steps` exact steps of a complex128 n1 x n2 x n3 state (reference: kron.step,
 * kron.py:110-121, applied `steps` times) with every two consecutive steps as
 * three fused launches: the first two products of step s per i3-plane
 * (mumode_plane12_kernel), the third products of steps s and s+1 together per
 * block of 32 fibers (mumode_pencil33_kernel: two E3 products on one
 * shared-memory tile), and the first two products of step s+1 per i3-plane.
 * Step s+1 therefore applies its directions in the order 3, 1, 2; products
 * along different directions commute, so the result differs from the
 * step-by-step order only in rounding.  An odd last step is (1,2) + 3.
 * E1..E3 row-major complex128 n_mu x n_mu; n1, n2, n3 in {32, 48, 64};
 * u is read, the result lands in out, ws is one state-sized scratch buffer
 * (u, out, ws must not alias).  Every launch is an ordinary stream launch, so
 * the call can be captured into a CUDA graph.
 */
int km_steps_paired(const void* u, const void* E1, const void* E2, const void* E3, int64_t n1, int64_t n2,
                    int64_t n3, int64_t steps, void* out, void* ws, void* stream);

/* bytes each of ws0/ws1 needs for km_tucker with these arguments */
int km_tucker_workspace(int u_dtype, int d, const int64_t* dims, const void* const* mats,
                        const int* mat_dtypes, const int64_t* rows, size_t* bytes);

/* standalone pointwise operator, out = op(in) over n elements of a complex
 * tensor (dtype KM_C64 or KM_C128); in == out is allowed */
int km_pointwise(const void* in, void* out, int dtype, int64_t n, const km_pointop* op,
                 void* stream);

/* km_pointwise with a widening store: in_dtype KM_C64 -> out_dtype KM_C128
 * (or equal dtypes; not in place when widening).  The op is evaluated as
 * numpy evaluates it on a state of in_dtype: for a complex64 state the GPE
 * density's squares and sum are float32 operations (psi.real**2 +
 * psi.imag**2, problems.py:543) before the float64 division by the weight
 * product, and the result is complex128 (the complex128 phase factor
 * promotes it, problems.py:545).  op == NULL / KM_OP_NONE is a plain cast. */
int km_pointwise_cast(const void* in, int in_dtype, void* out, int out_dtype, int64_t n,
                      const km_pointop* op, void* stream);

/*
 * Norms of a - b (b may be NULL) over n elements, result written to the
 * device double *result (reference: tensor.norm, tensor.py:169-198, and
 * relative_error, problems.py:160-169).  kind: 0 = max |.|, 1 = two-norm,
 * 2 = weighted two-norm with the weight product of a KM_OP_GPE_PHASE-style
 * km_pointop (weights[d-1] and inner_weights, dims).  Deterministic: fixed
 * grid, fixed reduction order.  workspace >= km_norm_workspace_bytes().
 */
size_t km_norm_workspace_bytes(void);
int km_norm(const void* a, const void* b, int dtype, int64_t n, int kind, const km_pointop* weights,
            double* result, void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KMB200_H */
