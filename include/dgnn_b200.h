/*
 * dgnn_b200.h -- C ABI of libdgnn_b200.so, the sm_100a kernels behind the
 * snapshot-sequence dynamic-GNN training hot path (arXiv 2109.07893).
 *
 * The reference (`dtgnn` 0.1.0, pure numpy) has no FFI; these entry points
 * are the ones its Python layer would bind for the hot path.
 * Each declaration cites the reference function it replaces.  Conventions:
 *   - plain device pointers and sizes, no torch types; all memory (including
 *     workspaces) is owned by the caller;
 *   - every call takes the cudaStream_t (as void*) it is enqueued on and is
 *     re-entrant (no hidden globals except the thread-local error string);
 *   - return 0 on success, a DGNN_E* code otherwise; dgnn_last_error() gives
 *     the message of the last failure on the calling thread;
 *   - data-dependent validation (corrupt deltas) is counted on device into a
 *     caller-provided int32 status word, read back when the caller chooses.
 * fp32 is the training arithmetic; graph values (Laplacian, first-layer
 * products) are computed in fp64 with IEEE-rounded ops (no FMA contraction)
 * so they equal the reference bit-for-bit before the fp32 downcast.
 */
#ifndef DGNN_B200_H
#define DGNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGNN_OK 0
#define DGNN_EINPUT 1        /* maps to InputError            */
#define DGNN_ECORRUPT 2      /* maps to CorruptDeltaError     */
#define DGNN_ECUDA 3         /* kernel launch / runtime error */
#define DGNN_EWORKSPACE 4    /* workspace too small           */
#define DGNN_EUNSUPPORTED 5  /* width outside the compiled set */

/* Row-addressed dense frame.  Row i lives at
 *   ptr + (i / rows_per_slab) * slab_stride + (i % rows_per_slab) * ld
 * (elements).  rows_per_slab == number of rows means a plain row-major
 * matrix.  The split form is the snapshot-owner layout of the multi-GPU
 * engine: [dest vertex chunk][owned step][rows of the chunk][width], which
 * NCCL all-to-all sends/receives without any pack/unpack copy. */
typedef struct {
    void* ptr;
    int64_t ld;
    int64_t rows_per_slab;
    int64_t slab_stride;
} dgnn_frame;

const char* dgnn_last_error(void);
int dgnn_abi_version(void);
/* Number of kernels launched through this library so far (process-wide). */
long long dgnn_launch_count(void);
/* Keep `sms` SMs free of the persistent (one CTA per SM) kernels so that
 * communication kernels running concurrently on another stream (NCCL P2P of
 * the multi-GPU exchange) are scheduled at once; 0 (default) uses all 148. */
void dgnn_set_sm_reserve(int sms);
/* 1 if the loaded cubin targets sm_100a and a device of that class is present */
int dgnn_device_check(int device);

/* ---------------- graph materialisation (K1/K2) ------------------------ */

/* CSR row pointer from a (row-)sorted COO row array:
 * rowptr[r] = lower_bound(rows, r), r in [0, n].  Used for full snapshots
 * (sorted u32 pairs, reference charge_full `delta.py:75-78`) and to index
 * delta pair lists. */
int dgnn_rowptr_from_sorted_rows(int32_t n, int64_t nnz, const int32_t* rows,
                                 int32_t* rowptr, void* stream);

size_t dgnn_csr_apply_delta_workspace(int32_t n);
/* K1 -- reference `delta.apply` (delta.py:126-146): new structure =
 * (old \ ext_prev) U ext_next, per-row merge in canonical column order.
 * del/ins are (row, col) pairs sorted lexicographically.  Validation as in
 * the reference: every ext_prev entry must exist in old, no ext_next entry
 * may collide with a kept entry; violations are counted into status[0].
 * Writes new_rowptr[n+1] and new_col[new_nnz]; new_cap bounds new_col. */
int dgnn_csr_apply_delta(int32_t n, const int32_t* old_rowptr, const int32_t* old_col,
                         int64_t n_del, const int32_t* del_row, const int32_t* del_col,
                         int64_t n_ins, const int32_t* ins_row, const int32_t* ins_col,
                         int32_t* new_rowptr, int32_t* new_col, int64_t new_cap,
                         void* workspace, size_t workspace_bytes, int32_t* status,
                         void* stream);

size_t dgnn_csr_transpose_workspace(int32_t n);
/* Deterministic CSR -> CSC (rows ascending inside each column, whatever
 * order the atomic scatter produced), carrying optional fp64 values.  Needed
 * for spmm_transpose (core.py:155-161) as a gather.  stage_col/stage_val are
 * caller scratch of nnz entries (stage_val only when val != NULL). */
int dgnn_csr_transpose_staged(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* col,
                              const double* val, int32_t* t_rowptr, int32_t* t_col, double* t_val,
                              int32_t* stage_col, double* stage_val, void* workspace,
                              size_t workspace_bytes, void* stream);

size_t dgnn_laplacian_workspace(int32_t n);
/* K2 -- reference `normalize_laplacian` (dtdg.py:178-191):
 * out = D^-1/2 (M + I) D^-1/2 restricted to the structure of M (+ diagonal),
 * D = 1 + out-degree of A taken from a_rowptr.  transposed = 0: M = A (CSR);
 * transposed = 1: M = A^T given as the CSC of A, producing the CSR of
 * Ahat^T.  val == NULL means unit values (value-free deltas).  Values are
 * (a * is_row(A)) * is_col(A) in fp64 without contraction; the diagonal is
 * fl(A-term + identity-term); exact zeros are elided (core.py:80).  Writes
 * out_rowptr[n+1], out_col, out_val32 and, if non-NULL, out_val64. */
int dgnn_laplacian(int32_t n, const int32_t* a_rowptr, const int32_t* m_rowptr,
                   const int32_t* m_col, const double* m_val, int transposed,
                   int32_t* out_rowptr, int32_t* out_col, float* out_val32, double* out_val64,
                   int64_t out_cap, void* workspace, size_t workspace_bytes, void* stream);

/* Degree features (dtdg.py:255-266): x[i] = (outdeg, indeg) as fp64
 * rows of width ld (>= 2). */
int dgnn_degree_features(int32_t n, const int32_t* rowptr, const int32_t* t_rowptr,
                         double* x, int64_t ld, void* stream);

/* M-smoothing of the snapshot sequence, window 2 (TM-GCN preprocessing on
 * the device; replaces `m_transform_graph` -> `sparse_weighted_sum`,
 * dtdg.py:239-252, core.py:173-192): out = wa A + wb B as a canonical CSR
 * with fp64 values, fl(fl(wa a) + fl(wb b)) where both hold the entry (the
 * reference's ascending-k np.add.at order), bit-identical.  val_a / val_b
 * may be NULL (unit values).  out_cap >= nnz_a + nnz_b. */
size_t dgnn_csr_weighted_merge_workspace(int32_t n, int64_t nnz_b);
int dgnn_csr_weighted_merge(int32_t n, const int32_t* rp_a, const int32_t* col_a, const double* val_a,
                            int64_t nnz_a, double wa, const int32_t* rp_b, const int32_t* col_b,
                            const double* val_b, int64_t nnz_b, double wb, int32_t* out_rowptr,
                            int32_t* out_col, double* out_val, int64_t out_cap, void* ws, size_t ws_bytes,
                            void* stream);

/* ---------------- sparse products (K3/K4) ------------------------------ */

/* Reference `spmm` (core.py:142-152) in fp64, sequential per row in
 * canonical order without FMA: bit-identical to np.add.at.  Called with the
 * CSC (CSR of A^T) it is `spmm_transpose` (core.py:155-161). */
int dgnn_spmm_f64(int32_t n, const int32_t* rowptr, const int32_t* col, const double* val,
                  const double* x, int64_t ldx, int32_t f, double* out, int64_t ldo,
                  void* stream);

/* fp32 SpMM out = M * x, M given as CSR (use the Ahat^T CSR for the
 * transpose product).  f in {4,16,32,64,128}. */
int dgnn_spmm_f32(int32_t n, const int32_t* rowptr, const int32_t* col, const float* val,
                  dgnn_frame x, int32_t f, dgnn_frame out, void* stream);

/* K3 -- fused graph convolution (training.py:342-357, models.py:200-212):
 *   s = (rowptr ? Ahat * x : x)     [fp widths, padded]
 *   q = s * w                       [w: fp x hp row-major]
 *   skip:  r = relu([s, q])  (width fp + hp)        (cd-gcn)
 *   plain: r = relu(q)       (width hp)             (tm-gcn)
 * s_out (nullable) keeps s for the backward.  fp in {4,16,32,64,128}
 * (4 only without aggregation), hp in {16,32,64,128}.  fp, hp <= 64 (fp >= 16)
 * run the tcgen05 instance (gather warps + 3xTF32 transform), the rest the
 * SIMT kernel. */
int dgnn_gcn_forward(int32_t n, const int32_t* rowptr, const int32_t* col, const float* val,
                     dgnn_frame x, int32_t fp, const float* w, int32_t hp, int skip,
                     dgnn_frame s_out, dgnn_frame r_out, void* stream);

/* Selects the K3 instance: 1 (default) tcgen05 where available, 0 SIMT. */
void dgnn_set_gcn_tensor_cores(int on);

/* K4 row part (training.py:347-350, 359-367):
 *   dpre = dr (.) [r > 0];  skip: ds = dpre[:, :fp] + dpre[:, fp:] * w^T
 *                           plain: ds = dpre * w^T                         */
int dgnn_gcn_backward_rows(int32_t n, dgnn_frame dr, dgnn_frame r, int32_t fp,
                           const float* w, int32_t hp, int skip, dgnn_frame ds, void* stream);

size_t dgnn_gcn_weight_grad_workspace(int32_t fp, int32_t hp);
/* K4 weight part: gw[k][j] += sum_i s[i][k] * dr[i][off + j] * [r[i][off + j] > 0]
 * (off = fp for skip, 0 for plain) -- deterministic split-K, fp64 final sum
 * accumulated into gw (fp x hp, fp64). */
int dgnn_gcn_weight_grad(int32_t n, dgnn_frame s, dgnn_frame dr, dgnn_frame r, int32_t fp,
                         int32_t hp, int skip, double* gw, void* workspace,
                         size_t workspace_bytes, void* stream);

/* ---------------- temporal stage (K5/K6/K7) ----------------------------- */

/* Cache layouts.  x, h (h_prev, h_out), dy, dh and dx are row-major.  The
 * per-step caches c (c_prev, c_out, c_new), gates / dz and dc are
 * TILE-BLOCKED over the step's `rows`: element (r, j) of an n x w array is
 * at  (r & ~127) w + (j / 4) 4 tr + (r & 127) 4 + (j % 4),
 * tr = min(128, n - (r & ~127))  -- 4-column groups of 128-row tiles stored
 * contiguously, so each warp access of these caches is 512 contiguous bytes.
 * A step's array occupies exactly n w floats.  dgnn_tile_block /
 * dgnn_tile_unblock convert. */

/* row-major (steps x n) x w  <->  tile-blocked per step of n rows */
int dgnn_tile_block(int64_t steps, int64_t n, int32_t w, const float* src, float* dst, void* stream);
int dgnn_tile_unblock(int64_t steps, int64_t n, int32_t w, const float* src, float* dst, void* stream);

/* K5 -- one LSTM step over `rows` vertex rows (training.py:370-391):
 *   z = [x | h_prev] * wcat + b,  wcat: (kx + hp) x 4hp, gate blocks [i|f|o|g]
 *   c = f c_prev + i g,  h = o tanh(c)
 * x rows have kx (= padded fin) columns at stride ldx; h rows stride hp;
 * c_prev / c_out tile-blocked (rows x hp); gates (nullable) caches [i|f|o|g],
 * tile-blocked rows x 4hp.  hp in {16,32,64,128}. */
int dgnn_lstm_forward_step(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                           const float* h_prev, const float* c_prev, const float* wcat,
                           const float* bias, float* h_out, float* c_out, float* gates,
                           void* stream);

/* Tensor-core operand image of a K-major weight matrix w (n x k, leading
 * dimension ldw): per 16-wide K chunk, the tf32 hi and lo parts
 * (hi = rna_tf32(w), lo = w - hi) as SWIZZLE_64B tiles, byte-identical to
 * their shared-memory copies.  n must be a multiple of 16 (<= 512). */
size_t dgnn_tc_weight_image_bytes(int32_t n, int32_t k);
int dgnn_tc_weight_image(int32_t n, int32_t k, const float* w, int64_t ldw, float* img, void* stream);
/* General form: n_alloc image rows of which the first n_valid come from w
 * (the rest zero); perm_hp > 0 takes the K order unit-major, element k
 * reading column (k % 4) * perm_hp + k / 4 (the backward-step operand). */
int dgnn_tc_weight_image_ex(int32_t n_alloc, int32_t n_valid, int32_t k, const float* w, int64_t ldw,
                            int32_t perm_hp, float* img, void* stream);

/* Self-test of the tcgen05 3xTF32 mainloop: d[m x n] = a[m x k] * w^T with
 * w given by its image (n in {64, 128, 256}). */
int dgnn_tc_gemm_test(int32_t m, int32_t n, int32_t k, const float* a, int64_t lda, const float* img,
                      float* d, int64_t ldd, void* stream);

/* K5 on tcgen05: same contract as dgnn_lstm_forward_step, the gate GEMM on
 * the tensor cores (kind::tf32, 3xTF32 = fp32-accurate, accumulator in TMEM)
 * with the cell update as the TMEM epilogue.  wimg = image of wcat^T
 * (4hp x (kx+hp)) from dgnn_tc_weight_image. */
int dgnn_lstm_forward_step_tc(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                              const float* h_prev, const float* c_prev, const float* wimg,
                              const float* bias, float* h_out, float* c_out, float* gates,
                              void* stream);

/* Persistent, warp-specialised versions (producer warps -> one MMA thread ->
 * epilogue warps, 4-stage smem ring, double-buffered TMEM accumulator; one
 * CTA per SM).  Same contracts and operand images as the _tc entries;
 * hp in {16, 32, 64}. */
/* K5 on CTA pairs (tcgen05.mma.cta_group::2, 2-CTA clusters): same contract
 * and bitwise the same results as dgnn_lstm_forward_step_ws; each CTA stages
 * its 128 rows and half of the weight chunk (hp 32 or 64). */
int dgnn_lstm_forward_step_pair(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                                const float* h_prev, const float* c_prev, const float* wimg, const float* bias,
                                float* h_out, float* c_out, float* gates, void* stream);
int dgnn_lstm_forward_step_ws(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                              const float* h_prev, const float* c_prev, const float* wimg,
                              const float* bias, float* h_out, float* c_out, float* gates,
                              void* stream);
int dgnn_lstm_backward_step_ws(int64_t rows, int32_t kx, int32_t hp, const float* dy,
                               const float* dh_in, const float* dc_in, float* gates,
                               const float* c_prev, const float* c_new, const float* wimg, float* dx,
                               int64_t lddx, float* dh_out, float* dc_out, void* stream);

/* K6 on tcgen05: same contract as dgnn_lstm_backward_step (dz written in
 * place of the gate cache `gates`); the pointwise gate gradients are the
 * operand producer of [dx | dh] = dz W^T (3xTF32, TMEM accumulator).
 * wimg = dgnn_tc_weight_image_ex(round16(kx+hp), kx+hp, 4hp, wcat, 4hp,
 * hp, ...).  hp in {16, 32, 64} with kx + hp <= 256. */
int dgnn_lstm_backward_step_tc(int64_t rows, int32_t kx, int32_t hp, const float* dy,
                               const float* dh_in, const float* dc_in, float* gates,
                               const float* c_prev, const float* c_new, const float* wimg, float* dx,
                               int64_t lddx, float* dh_out, float* dc_out, void* stream);

/* LSTM weight gradients of a whole block on tcgen05 (training.py:422-424):
 *   gwcat[k][j] += sum_r xcat[r][k] dz[r][j],  gb[j] += sum_r dz[r][j]
 * over rows r = t*np + v of the block (rows = bsize*np), with
 * xcat[r] = [x[r] (kx cols, ld ldx) | h_prev] and h_prev = h_out[r - np]
 * (t > 0) or h0[v] (t = 0).  dz: bsize steps of np x 4hp, each tile-blocked
 * (the backward step's in-place output).  Operands MN-major straight
 * from HBM, 3xTF32, TMEM accumulation restarted every 512 rows and promoted
 * to per-CTA fp32 slots, fp64 fixed-order final reduction.  hp in
 * {32, 64}, kx + hp <= 256. */
size_t dgnn_lstm_weight_grad_tc_workspace(int32_t kx, int32_t hp);
int dgnn_lstm_weight_grad_tc(int64_t rows, int64_t np, int32_t kx, int32_t hp, const float* x,
                             int64_t ldx, const float* h_out, const float* h0, const float* dz,
                             double* gwcat, double* gb, void* workspace, size_t workspace_bytes,
                             void* stream);
/* Same product with the dz operand staged in TMEM (tcgen05 A-from-TMEM MMAs;
 * shared memory carries xcat only).  Same arguments and workspace
 * (dgnn_lstm_weight_grad_tc_workspace); results agree to the accumulation
 * order of the products. */
int dgnn_lstm_weight_grad_ts(int64_t rows, int64_t np, int32_t kx, int32_t hp, const float* x,
                             int64_t ldx, const float* h_out, const float* h0, const float* dz,
                             double* gwcat, double* gb, void* workspace, size_t workspace_bytes,
                             void* stream);

/* K6 -- one reverse LSTM step (training.py:404-426):
 *   dh = dy + dh_in; do, dc, df, di, dg as the reference; dc_out = dc f
 *   dz = [di i(1-i) | df f(1-f) | do o(1-o) | dg (1-g^2)]  (written, 4hp wide)
 *   [dx | dh_out] = dz * wcat^T   using wcat_t (4hp x (kx+hp), row-major)
 * dy == NULL means zero.  dz may alias gates (in-place).  gates, dz, c_prev,
 * c_new, dc_in, dc_out tile-blocked; dy, dh_in, dh_out, dx row-major. */
int dgnn_lstm_backward_step(int64_t rows, int32_t kx, int32_t hp, const float* dy,
                            const float* dh_in, const float* dc_in, const float* gates,
                            const float* c_prev, const float* c_new, const float* wcat_t,
                            float* dz, float* dx, int64_t lddx, float* dh_out, float* dc_out,
                            void* stream);

size_t dgnn_gemm_tn_workspace(int32_t m, int32_t n);
/* Deterministic split-K weight-gradient GEMM: out[m][n] += sum_r a[r][m] b[r][n]
 * (the x^T dz, h^T dz products of training.py:422-424), fp32 partials,
 * fixed-order fp64 reduction into out (ld = ldo).  If colsum != NULL also
 * colsum[n] += sum_r b[r][n] (the db of training.py:424). */
int dgnn_gemm_tn(int64_t rows, int32_t m, int32_t n, const float* a, int64_t lda,
                 const float* b, int64_t ldb, double* out, int64_t ldo, double* colsum,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Banded frame combinations in one launch (the M-product forward / adjoint,
 * training.py:430-460): for i < nout, out_i = [out_i +] sum_j tcoef[j] *
 * tsrc[j] over j in [tptr[i], tptr[i+1]) in order (each product rounded,
 * then added: dgnn_axpy_frame's arithmetic).  outs / tsrc hold device
 * addresses of fp32 frames of `count` floats (a multiple of 4); accum[i] = 1
 * adds onto the existing out_i.  Outputs are produced in order, so an
 * output may read frames written by earlier outputs of the same call. */
int dgnn_frames_combine(int64_t count, int32_t nout, const int64_t* outs, const int32_t* accum, const int32_t* tptr,
                        const int64_t* tsrc, const float* tcoef, void* stream);
/* K7 -- banded M-product term (training.py:430-441): z = coef * y (init=1)
 * or z += coef * y (init=0), over rows x width contiguous fp32. */
int dgnn_axpy_frame(int64_t count, float coef, const float* y, float* z, int init, void* stream);

/* ---------------- head / loss (K8) -------------------------------------- */

/* Link-prediction head + softmax CE (models.py:335-348, training.py:102-126,
 * 698-735) for one frame:
 *   logits_p = z[u_p] . hw[:E] + z[v_p] . hw[E:] + hb   (hw: 2*ep x c, rows
 *              [0,E) and [ep, ep+E) real)
 *   loss_per_pair[p] = CE_p in fp64 (sum it with dgnn_sum_f64)
 *   dlogits_p = (softmax - onehot) * scale in fp64 (if dlogits != NULL): the
 *   head reductions stay fp64 so exact cancellations (e.g. the bias gradient
 *   of a balanced label set) stay ~0 as in the reference, which Adam's
 *   g / (|g| + eps) would otherwise amplify */
int dgnn_head_loss(int64_t npairs, const int32_t* u, const int32_t* v, const int32_t* y,
                   dgnn_frame z, int32_t ep, int32_t c, const float* hw, const float* hb,
                   double scale, double* loss_per_pair, int32_t n_loss, double* dlogits,
                   void* stream);

/* Head parameter grads: ghw[k][j] += sum_p cat_p[k] dlogits_p[j], ghb += sum_p dlogits_p
 * (deterministic split + fp64 reduce).  Workspace from dgnn_head_grad_workspace. */
size_t dgnn_head_grad_workspace(int32_t ep, int32_t c);
int dgnn_head_grad(int64_t npairs, const int32_t* u, const int32_t* v, dgnn_frame z, int32_t ep,
                   int32_t c, const double* dlogits, double* ghw, double* ghb, void* workspace,
                   size_t workspace_bytes, void* stream);

/* K8 fused (training.py:698-735, 2 classes): head_loss and head_grad in one
 * pass over the pairs -- loss_pp and dlogits as dgnn_head_loss, ghw / ghb
 * accumulated as dgnn_head_grad (deterministic fixed-order reduction).
 * Workspace from dgnn_head_grad_workspace. */
int dgnn_head_loss_grad(int64_t npairs, const int32_t* u, const int32_t* v, const int32_t* y, dgnn_frame z,
                        int32_t ep, int32_t c, const float* hw, const float* hb, double scale, double* loss_pp,
                        int32_t n_partials, double* dlogits, double* ghw, double* ghb, void* ws, size_t ws_bytes,
                        void* stream);
/* dz seeds (training.py:732-734) as a gather over the vertex->slot
 * incidence (ascending slot order = the np.add.at order):
 *   dz[x] = sum_{slot s of x} dlogits[s/2] . hw[side(s)]^T ; zero rows elsewhere. */
int dgnn_head_scatter(int32_t n, const int32_t* inc_ptr, const int32_t* inc_slot,
                      const double* dlogits, const float* hw, int32_t ep, int32_t c,
                      dgnn_frame dz, void* stream);
/* Same seeds with the list of vertices that have incident pairs
 * (`active`, ascending, n_active of them): rows without pairs are
 * zero-filled by a flat pass and only the active rows are gathered
 * (bit-identical to dgnn_head_scatter). */
int dgnn_head_scatter_active(int32_t n, const int32_t* inc_ptr, const int32_t* inc_slot, int32_t n_active,
                             const int32_t* active, const double* dlogits, const float* hw, int32_t ep, int32_t c,
                             dgnn_frame dz, void* stream);

/* Test accuracy (training.py:189-197): *correct += #pairs whose first-index
 * argmax of the logits equals the label (int64 counter, integer atomics). */
int dgnn_head_predict(int64_t npairs, const int32_t* u, const int32_t* v, const int32_t* y,
                      dgnn_frame z, int32_t ep, int32_t c, const float* hw, const float* hb,
                      int64_t* correct, void* stream);

/* Deterministic sum of fp64 values into *out (out = sum, or += if
 * accumulate): one 8-CTA cluster, summation order fixed by n alone. */
int dgnn_sum_f64(int64_t n, const double* x, double* out, int accumulate, void* stream);

/* ---------------- parameters / optimiser (K9) --------------------------- */

/* Adam in fp64 over a flat buffer (training.py:886-900), IEEE-rounded ops
 * in the reference's evaluation order.  The scalars are passed exactly as the
 * reference forms them in Python: one_m_beta = 1.0 - beta, bc = 1.0 - beta**t. */
int dgnn_adam(int64_t n, double* p, const double* g, double* m, double* v, double lr, double beta1,
              double one_m_beta1, double beta2, double one_m_beta2, double bc1, double bc2, double eps,
              void* stream);
/* w32[pos0[i]] = (float)p[i]; w32[pos1[i]] = (float)p[i] when pos1[i] >= 0 */
int dgnn_params_to_device(int64_t n, const double* p, const int64_t* pos0, const int64_t* pos1,
                          float* w32, void* stream);
/* g[i] = gpad[pos0[i]] */
int dgnn_grads_gather(int64_t n, const double* gpad, const int64_t* pos0, double* g,
                      void* stream);

/* out[pos[i]] = p[i] (fp64 padded image of the master parameters) */
int dgnn_scatter_f64(int64_t n, const double* p, const int64_t* pos, double* out, void* stream);

/* EGCN-O weight evolution (egcn_evolve, models.py:247-268; evolve chain,
 * training.py:466-509), elementwise over cnt (padded F x H) weights, fp64,
 * `steps` timesteps of a block.  Forward: from w_in, writes the final weight
 * to w_out, every step's weight as fp32 to images[s * cnt ...] and (if
 * non-NULL) the per-step cache [w_prev | i | f | o | g | tanh c] to
 * cache[s * 6 cnt ...].  Backward: seeds[s * cnt ...] = dL/dW_s (NULL: none),
 * dw_carry in = gradient w.r.t. the block's final weight, out = w.r.t. its
 * input weight; dgates / dbias (4 cnt each) += the block's gate gradients. */
int dgnn_evolve_forward(int64_t cnt, int32_t steps, const double* gates, const double* bias, const double* w_in,
                        double* w_out, float* images, double* cache, void* stream);
int dgnn_evolve_backward(int64_t cnt, int32_t steps, const double* gates, const double* cache,
                         const double* seeds, double* dw_carry, double* dgates, double* dbias, void* stream);

/* Elementwise helpers for frame plumbing. */
int dgnn_fill_f32(int64_t n, float value, float* x, void* stream);
int dgnn_cast_f64_to_f32_frame(int32_t n, int32_t f, const double* x, int64_t ldx,
                               dgnn_frame out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DGNN_B200_H */
