// Deterministic weight-gradient reductions and small dense helpers.
//
// Weight gradients in the reference are sums over every vertex row of
// every timestep (training.py:365, 422-424, 730-731).  Here they are split-K
// GEMMs: CTA (tile, chunk) accumulates a 64x64 fp32 partial over a fixed row
// range in registers (4x4 per thread), partials are reduced in a fixed order
// in fp64 and added to an fp64 gradient accumulator -- bit-reproducible from
// run to run, no floating-point atomics anywhere.
#include "common.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace dgnn {

constexpr int TN_BM = 64, TN_BN = 64, TN_BR = 16;

// tcgen05 GCN weight gradient (gcn_dw_tc.cu) and the K3/K4 engine switch (spmm.cu)
size_t gcn_dw_tc_workspace(int fp, int hp);
int gcn_dw_tc(int32_t n, dgnn_frame s, dgnn_frame dr, dgnn_frame r, int fp, int hp, int skip, double* gw, void* ws,
              size_t ws_bytes, cudaStream_t st);
int gcn_tensor_cores_on();

// Loaders map (row r, column c) of the logical A / B operands to memory; c is
// always a multiple of 4 and the 4 columns are contiguous.
struct PlainLoader {
    const float* p;
    int64_t ld;
    int ncols;
    __device__ __forceinline__ float4 load(int64_t r, int c) const {
        if (c >= ncols) return make_float4(0.f, 0.f, 0.f, 0.f);
        return *reinterpret_cast<const float4*>(p + r * ld + c);
    }
};

struct FrameLoader {
    dgnn_frame f;
    int off, ncols;
    __device__ __forceinline__ float4 load(int64_t r, int c) const {
        if (c >= ncols) return make_float4(0.f, 0.f, 0.f, 0.f);
        return *reinterpret_cast<const float4*>(frame_row<const float>(f, r) + off + c);
    }
};

// dq = dr[off + c] * [r[off + c] > 0]
struct MaskedFrameLoader {
    dgnn_frame dr, r;
    int off, ncols;
    __device__ __forceinline__ float4 load(int64_t row, int c) const {
        if (c >= ncols) return make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 g = *reinterpret_cast<const float4*>(frame_row<const float>(dr, row) + off + c);
        const float4 m = *reinterpret_cast<const float4*>(frame_row<const float>(r, row) + off + c);
        return make_float4(m.x > 0.f ? g.x : 0.f, m.y > 0.f ? g.y : 0.f, m.z > 0.f ? g.z : 0.f,
                           m.w > 0.f ? g.w : 0.f);
    }
};

// partial[chunk][m][n] = sum_{r in chunk} A[r][m] * B[r][n]   (64x64 tile per CTA)
// colsum partial (row m = M) when with_colsum: sum_r B[r][n].
template <typename LA, typename LB>
__global__ void __launch_bounds__(256) tn_partial_kernel(int64_t rows, int M, int N, LA la, LB lb,
                                                         int64_t rows_per_chunk, float* __restrict__ part,
                                                         int ldp, int with_colsum) {
    __shared__ __align__(16) float As[TN_BR][TN_BM];
    __shared__ __align__(16) float Bs[TN_BR][TN_BN];
    const int tiles_n = (N + TN_BN - 1) / TN_BN;
    const int tile = blockIdx.x, chunk = blockIdx.y;
    const int m0 = (tile / tiles_n) * TN_BM, n0 = (tile % tiles_n) * TN_BN;
    const int tid = threadIdx.x, tm = tid / 16, tn = tid % 16;
    const int64_t r0 = chunk * rows_per_chunk;
    const int64_t r1 = min(rows, r0 + rows_per_chunk);
    float acc[4][4];
    float csum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    const int lr = tid / 16, lc = (tid % 16) * 4;  // loader: row lr of the 16-row stage, 4 columns
    for (int64_t rb = r0; rb < r1; rb += TN_BR) {
        const int64_t r = rb + lr;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (r < r1) {
            a = la.load(r, m0 + lc);
            b = lb.load(r, n0 + lc);
        }
        *reinterpret_cast<float4*>(&As[lr][lc]) = a;
        *reinterpret_cast<float4*>(&Bs[lr][lc]) = b;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TN_BR; ++k) {
            const float4 av = *reinterpret_cast<const float4*>(&As[k][4 * tm]);
            const float4 bv = *reinterpret_cast<const float4*>(&Bs[k][4 * tn]);
            const float x[4] = {av.x, av.y, av.z, av.w}, y[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(x[i], y[j], acc[i][j]);
            if (with_colsum && tm == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) csum[j] += y[j];
            }
        }
        __syncthreads();
    }
    float* out = part + (int64_t)chunk * ldp * (M + 1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + 4 * tm + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + 4 * tn + j;
            if (n < N) out[(int64_t)m * ldp + n] = acc[i][j];
        }
    }
    if (with_colsum && tm == 0 && m0 == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + 4 * tn + j;
            if (n < N) out[(int64_t)M * ldp + n] = csum[j];
        }
    }
}

// out[m][n] += sum_chunk part[chunk][m][n]  (fp64, ascending chunk order)
__global__ void tn_reduce_kernel(int M, int N, int nchunks, const float* __restrict__ part, int ldp,
                                 double* __restrict__ out, int64_t ldo, double* __restrict__ colsum) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)(M + (colsum ? 1 : 0)) * N;
    if (i >= total) return;
    const int m = (int)(i / N), n = (int)(i % N);
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += (double)part[((int64_t)c * (M + 1) + m) * ldp + n];
    if (m < M) out[(int64_t)m * ldo + n] += s;
    else colsum[n] += s;
}

constexpr int kMaxChunks = 2 * kMaxSMs;

static int chunks_for(int64_t rows, int tiles) {
    int64_t c = cdiv(2 * num_sms(), tiles);             // ~2 CTAs per SM in total
    const int64_t by_rows = cdiv(rows, 4 * TN_BR);  // at least 64 rows per chunk
    if (c > by_rows) c = by_rows;
    if (c < 1) c = 1;
    if (c > kMaxChunks) c = kMaxChunks;
    return (int)c;
}

size_t tn_workspace_bytes(int M, int N) {
    return (size_t)kMaxChunks * (M + 1) * N * sizeof(float) + 256;
}

template <typename LA, typename LB>
int tn_run(int64_t rows, int M, int N, LA la, LB lb, double* out, int64_t ldo, double* colsum, void* ws,
           size_t ws_bytes, cudaStream_t st, const char* what) {
    if (rows <= 0 || M <= 0 || N <= 0) return DGNN_OK;
    if (ws_bytes < tn_workspace_bytes(M, N)) {
        set_error("%s: workspace too small", what);
        return DGNN_EWORKSPACE;
    }
    const int tiles = (int)(cdiv(M, TN_BM) * cdiv(N, TN_BN));
    const int nch = chunks_for(rows, tiles);
    const int64_t per = cdiv(cdiv(rows, nch), TN_BR) * TN_BR;
    const int nch_eff = (int)cdiv(rows, per);
    float* part = reinterpret_cast<float*>(ws);
    ::dgnn::note_launch();
    tn_partial_kernel<LA, LB><<<dim3(tiles, nch_eff), 256, 0, st>>>(rows, M, N, la, lb, per, part, N,
                                                                     colsum ? 1 : 0);
    const int64_t total = (int64_t)(M + (colsum ? 1 : 0)) * N;
    ::dgnn::note_launch();
    tn_reduce_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(M, N, nch_eff, part, N, out, ldo, colsum);
    return launch_status(what);
}

// deterministic fp64 sum, one 8-CTA cluster (8 SMs of load bandwidth; a
// single CTA was latency-bound at ~50 GB/s): thread g of the cluster keeps 8
// partial sums over x[g + k * 8192 + j * 65536] (8 loads in flight), combined
// by a fixed tree, then a fixed shuffle tree per warp, the 32 warp sums in
// order, and the 8 CTA sums read by CTA 0 over distributed shared memory in
// rank order.  The order depends only on n, never on the schedule.
constexpr int kSumCtas = 8;
__global__ void __cluster_dims__(kSumCtas, 1, 1) __launch_bounds__(1024)
    sum_f64_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ out, int accumulate) {
    __shared__ double wsum[32];
    __shared__ double csum;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    constexpr int64_t T = (int64_t)kSumCtas * 1024;
    double p[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int64_t i = (int64_t)rank * 1024 + threadIdx.x;
    for (; i + 7 * T < n; i += 8 * T) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = x[i + k * T];
#pragma unroll
        for (int k = 0; k < 8; ++k) p[k] += v[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (i + k * T < n) p[k] += x[i + k * T];
    double s = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = wsum[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
        if (threadIdx.x == 0) csum = w;
    }
    cl.sync();
    if (rank == 0 && threadIdx.x == 0) {
        double c[kSumCtas];
#pragma unroll
        for (int q = 0; q < kSumCtas; ++q) c[q] = *cl.map_shared_rank(&csum, q);
        const double t = ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7]));
        *out = accumulate ? (*out + t) : t;
    }
    cl.sync();   // keep every CTA's csum alive until CTA 0 has read it
}

__global__ void axpy_kernel(int64_t n, float coef, const float* __restrict__ y, float* __restrict__ z,
                            int init) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float t = __fmul_rn(coef, y[i]);
    z[i] = init ? t : __fadd_rn(z[i], t);
}

// Banded frame combinations in one pass (the M-product, training.py:430-460):
// out_i = [out_i +] sum_j c_ij * src_ij, terms in table order, each product
// rounded then added (the axpy sequence above, bitwise).  One thread per
// float4 of a frame runs every output in order, so a source frame shared by
// consecutive outputs is re-read from L1/L2, and an output may be a source
// of a LATER output (the table is built that way).
__global__ void frames_combine_kernel(int64_t n4, int nout, const int64_t* __restrict__ outs,
                                      const int32_t* __restrict__ accum, const int32_t* __restrict__ tptr,
                                      const int64_t* __restrict__ tsrc, const float* __restrict__ tcoef) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
        for (int i = 0; i < nout; ++i) {
            float4* out = reinterpret_cast<float4*>(outs[i]) + e;
            float4 acc = accum[i] ? *out : make_float4(0.f, 0.f, 0.f, 0.f);
            bool first = !accum[i];
            for (int j = tptr[i]; j < tptr[i + 1]; ++j) {
                const float4 v = reinterpret_cast<const float4*>(tsrc[j])[e];
                const float c = tcoef[j];
                const float4 t = make_float4(__fmul_rn(c, v.x), __fmul_rn(c, v.y), __fmul_rn(c, v.z), __fmul_rn(c, v.w));
                acc = first ? t : make_float4(__fadd_rn(acc.x, t.x), __fadd_rn(acc.y, t.y), __fadd_rn(acc.z, t.z),
                                              __fadd_rn(acc.w, t.w));
                first = false;
            }
            *out = acc;
        }
    }
}

// row-major <-> tile-blocked (common.cuh tb_off), one float per thread
template <bool TO_BLOCKED>
__global__ void tile_block_kernel(int64_t total, int64_t n, int w, const float* __restrict__ src,
                                  float* __restrict__ dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t step_elems = n * w;
    const int64_t t = i / step_elems, rem = i - t * step_elems;
    const int64_t r = rem / w;
    const int j = (int)(rem - r * w);
    const int64_t b = t * step_elems + tb_off(r, j, w, n);
    if (TO_BLOCKED) dst[b] = src[i];
    else dst[i] = src[b];
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

int dgnn_tile_block(int64_t steps, int64_t n, int32_t w, const float* src, float* dst, void* stream) {
    DGNN_CHECK_ARG(steps >= 0 && n >= 0 && w > 0 && w % 4 == 0, "tile_block: bad sizes");
    const int64_t total = steps * n * w;
    if (total == 0) return DGNN_OK;
    ::dgnn::note_launch();
    tile_block_kernel<true><<<(unsigned)cdiv(total, 256), 256, 0, as_stream(stream)>>>(total, n, w, src, dst);
    return launch_status("tile_block");
}

int dgnn_tile_unblock(int64_t steps, int64_t n, int32_t w, const float* src, float* dst, void* stream) {
    DGNN_CHECK_ARG(steps >= 0 && n >= 0 && w > 0 && w % 4 == 0, "tile_unblock: bad sizes");
    const int64_t total = steps * n * w;
    if (total == 0) return DGNN_OK;
    ::dgnn::note_launch();
    tile_block_kernel<false><<<(unsigned)cdiv(total, 256), 256, 0, as_stream(stream)>>>(total, n, w, src, dst);
    return launch_status("tile_unblock");
}

size_t dgnn_gemm_tn_workspace(int32_t m, int32_t n) { return tn_workspace_bytes(m, n); }

int dgnn_gemm_tn(int64_t rows, int32_t m, int32_t n, const float* a, int64_t lda, const float* b, int64_t ldb,
                 double* out, int64_t ldo, double* colsum, void* ws, size_t ws_bytes, void* stream) {
    DGNN_CHECK_ARG(m % 4 == 0 && n % 4 == 0 && lda % 4 == 0 && ldb % 4 == 0, "gemm_tn: widths must be x4");
    return tn_run(rows, m, n, PlainLoader{a, lda, m}, PlainLoader{b, ldb, n}, out, ldo, colsum, ws, ws_bytes,
                  as_stream(stream), "gemm_tn");
}

size_t dgnn_gcn_weight_grad_workspace(int32_t fp, int32_t hp) {
    const size_t a = tn_workspace_bytes(fp, hp), b = gcn_dw_tc_workspace(fp, hp);
    return a > b ? a : b;
}

int dgnn_gcn_weight_grad(int32_t n, dgnn_frame s, dgnn_frame dr, dgnn_frame r, int32_t fp, int32_t hp, int skip,
                         double* gw, void* ws, size_t ws_bytes, void* stream) {
    DGNN_CHECK_ARG(fp % 4 == 0 && hp % 4 == 0, "gcn_weight_grad: widths must be x4");
    if (n <= 0) return DGNN_OK;
    if (gcn_tensor_cores_on()) {
        const int rc = gcn_dw_tc(n, s, dr, r, fp, hp, skip, gw, ws, ws_bytes, as_stream(stream));
        if (rc >= 0) return rc;
    }
    const int off = skip ? fp : 0;
    return tn_run((int64_t)n, fp, hp, FrameLoader{s, 0, fp}, MaskedFrameLoader{dr, r, off, hp}, gw, hp, nullptr,
                  ws, ws_bytes, as_stream(stream), "gcn_weight_grad");
}

int dgnn_sum_f64(int64_t n, const double* x, double* out, int accumulate, void* stream) {
    ::dgnn::note_launch();
    sum_f64_kernel<<<kSumCtas, 1024, 0, as_stream(stream)>>>(n, x, out, accumulate);
    return launch_status("sum_f64");
}

int dgnn_frames_combine(int64_t count, int32_t nout, const int64_t* outs, const int32_t* accum, const int32_t* tptr,
                        const int64_t* tsrc, const float* tcoef, void* stream) {
    DGNN_CHECK_ARG(count % 4 == 0 && nout >= 0, "frames_combine: count must be a multiple of 4");
    if (count == 0 || nout == 0) return DGNN_OK;
    const int64_t n4 = count / 4;
    int64_t blocks = cdiv(n4, 256);
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    ::dgnn::note_launch();
    frames_combine_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(n4, nout, outs, accum, tptr, tsrc, tcoef);
    return launch_status("frames_combine");
}

int dgnn_axpy_frame(int64_t count, float coef, const float* y, float* z, int init, void* stream) {
    if (count == 0) return DGNN_OK;
    ::dgnn::note_launch();
    axpy_kernel<<<(unsigned)cdiv(count, 256), 256, 0, as_stream(stream)>>>(count, coef, y, z, init);
    return launch_status("axpy_frame");
}

}  // extern "C"
