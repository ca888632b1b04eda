// Sparse aggregation kernels (K3/K4): vectorised CSR SpMM with the dense
// GCN transform and activation fused into the epilogue, and the row part of
// the GCN backward.  Reference: core.py:142-161 (spmm / spmm_transpose),
// training.py:342-367 (plain / skip-concat GCN cells), models.py:200-212.
//
// Layout: a row group of G = F/4 lanes owns one CSR row; every lane holds a
// float4 slice of the aggregated row, so each gathered neighbour row is one
// fully coalesced F*4-byte read.  The dense transform reads W from shared
// memory and broadcasts the aggregated row across the group with shuffles.
#include "common.cuh"

namespace dgnn {

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 relu4(float4 v) {
    return make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
}
__device__ __forceinline__ void fma4(float4& a, float s, float4 b) {
    a.x = fmaf(s, b.x, a.x);
    a.y = fmaf(s, b.y, a.y);
    a.z = fmaf(s, b.z, a.z);
    a.w = fmaf(s, b.w, a.w);
}
__device__ __forceinline__ float comp(const float4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Row aggregation: acc = sum_e val[e] * x[col[e]][4gl .. 4gl+3], 4-way unrolled
// so four independent gathers are in flight per lane.
__device__ __forceinline__ float4 gather_row(int64_t row, const int32_t* __restrict__ rp,
                                             const int32_t* __restrict__ col,
                                             const float* __restrict__ val, const dgnn_frame& x,
                                             int gl) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int e = rp[row];
    int ee = rp[row + 1];
    if (ee - e > kHubRow) ee = e;   // hub rows: hub_rows_kernel
    for (; e + 3 < ee; e += 4) {
        const int c0 = __ldg(col + e), c1 = __ldg(col + e + 1), c2 = __ldg(col + e + 2),
                  c3 = __ldg(col + e + 3);
        const float v0 = __ldg(val + e), v1 = __ldg(val + e + 1), v2 = __ldg(val + e + 2),
                    v3 = __ldg(val + e + 3);
        const float4 x0 = ldg4(frame_row<const float>(x, c0) + 4 * gl);
        const float4 x1 = ldg4(frame_row<const float>(x, c1) + 4 * gl);
        const float4 x2 = ldg4(frame_row<const float>(x, c2) + 4 * gl);
        const float4 x3 = ldg4(frame_row<const float>(x, c3) + 4 * gl);
        fma4(acc, v0, x0);
        fma4(acc, v1, x1);
        fma4(acc, v2, x2);
        fma4(acc, v3, x3);
    }
    for (; e < ee; ++e) fma4(acc, __ldg(val + e), ldg4(frame_row<const float>(x, __ldg(col + e)) + 4 * gl));
    return acc;
}

template <int F>
__global__ void __launch_bounds__(256) spmm_f32_kernel(int32_t n, const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ col,
                                                       const float* __restrict__ val, dgnn_frame x,
                                                       dgnn_frame out) {
    constexpr int G = F / 4, RW = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = warp * RW + sub; row < n; row += nwarps * RW)
        st4(frame_row<float>(out, row) + 4 * gl, gather_row(row, rp, col, val, x, gl));
}

// Hub rows (degree > kHubRow) of an aggregation, after the main kernel on the
// same stream.  MODE 0: out = s (SpMM); 1: skip GCN r = [relu(s), relu(sW)]
// (+ s_out); 2: plain GCN r = relu(sW) (+ s_out).  Each CTA scans 256 rows
// at a time and computes each hub among them: G = F/4 lanes per edge slot,
// 256/G slots each summing a strided share of the edges in order, slots
// combined by a fixed tree; q_j = sum_k s_k W[k][j] in k order.
// edges of a CTA slot in flight per step on rows of more than kWarpHub entries
#ifndef DGNN_HUB_UB
#define DGNN_HUB_UB 8
#endif
template <int F, int H, int MODE>
__global__ void __launch_bounds__(256) hub_rows_kernel(int32_t n, const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ col,
                                                       const float* __restrict__ val, dgnn_frame x,
                                                       const float* __restrict__ w, dgnn_frame s_out,
                                                       dgnn_frame r_out) {
    // Rows of kHubRow+1..kWarpHub entries: a warp each (SL slots of G lanes,
    // slot sums combined by a fixed shuffle tree), several in flight per
    // CTA; longer rows: the whole CTA (EPS slots, fixed smem tree).  q_j =
    // sum_k s_k W[k][j] in k order.
    constexpr int G = F / 4, EPS = 256 / G, SL = 32 / G;
    constexpr int kWarpHub = 512;
    __shared__ int32_t list[256];
    __shared__ int cnt, nbig;
    __shared__ float4 part[EPS][G];
    __shared__ float4 wrow[8][G];   // a warp's row aggregate (the W product reads it)
    const int slot = threadIdx.x / G, gl = threadIdx.x % G;
    const int lane = threadIdx.x & 31, wslot = lane / G, wid = threadIdx.x >> 5;
    auto emit = [&](int row, const float4& s4, bool lead, int jlane, int jstride, const float* sk) {
        // s4: the row's aggregate (the G lead lanes hold F floats); sk: the same in shared memory
        if constexpr (MODE == 0) {
            if (lead) st4(frame_row<float>(r_out, row) + 4 * gl, s4);
        } else {
            float* rr = frame_row<float>(r_out, row);
            if (lead) {
                if (s_out.ptr) st4(frame_row<float>(s_out, row) + 4 * gl, s4);
                if (MODE == 1) st4(rr + 4 * gl, relu4(s4));
            }
            for (int j = jlane; j < H; j += jstride) {
                float q = 0.f;
                for (int kk = 0; kk < F; ++kk) q = fmaf(sk[kk], __ldg(w + kk * H + j), q);
                rr[(MODE == 1 ? F : 0) + j] = fmaxf(q, 0.f);
            }
        }
    };
    for (int64_t base = (int64_t)blockIdx.x * 256; base < n; base += (int64_t)gridDim.x * 256) {
        if (threadIdx.x == 0) cnt = 0, nbig = 0;
        __syncthreads();
        const int64_t r = base + threadIdx.x;
        if (r < n) {
            const int d = rp[r + 1] - rp[r];
            if (d > kWarpHub) list[255 - atomicAdd(&nbig, 1)] = (int32_t)r;
            else if (d > kHubRow) list[atomicAdd(&cnt, 1)] = (int32_t)r;
        }
        __syncthreads();
        const int nh = cnt, nb = nbig;
        // mid rows: warp wid takes rows wid, wid + 8, ...
        for (int k = wid; k < nh; k += 8) {
            const int row = list[k];
            const int eb = rp[row], ee = rp[row + 1];
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            int e = eb + wslot;
            for (; e + 7 * SL < ee; e += 8 * SL) {
                int c[8];
                float v[8];
                float4 xv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    c[j] = __ldg(col + e + j * SL);
                    v[j] = __ldg(val + e + j * SL);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) xv[j] = ldg4(frame_row<const float>(x, c[j]) + 4 * gl);
#pragma unroll
                for (int j = 0; j < 8; ++j) fma4(acc, v[j], xv[j]);
            }
            for (; e < ee; e += SL)
                fma4(acc, __ldg(val + e), ldg4(frame_row<const float>(x, __ldg(col + e)) + 4 * gl));
#pragma unroll
            for (int o = 16; o >= G; o >>= 1) {
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
                acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
            }
            if (lane < G) wrow[wid][gl] = acc;
            __syncwarp();
            emit(row, acc, lane < G, lane, 32, reinterpret_cast<const float*>(&wrow[wid][0]));
            __syncwarp();
        }
        // long rows: the whole CTA each
        for (int k = 0; k < nb; ++k) {
            const int row = list[255 - k];
            const int eb = rp[row], ee = rp[row + 1];
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            int e = eb + slot;
            // UB of the slot's edges in flight at once (a hub of ~8000 edges was a
            // 250-step chain of dependent col -> x loads)
            constexpr int UB = DGNN_HUB_UB;
            for (; e + (UB - 1) * EPS < ee; e += UB * EPS) {
                int c[UB];
                float v[UB];
                float4 xv[UB];
#pragma unroll
                for (int j = 0; j < UB; ++j) {
                    c[j] = __ldg(col + e + j * EPS);
                    v[j] = __ldg(val + e + j * EPS);
                }
#pragma unroll
                for (int j = 0; j < UB; ++j) xv[j] = ldg4(frame_row<const float>(x, c[j]) + 4 * gl);
#pragma unroll
                for (int j = 0; j < UB; ++j) fma4(acc, v[j], xv[j]);
            }
            for (; e < ee; e += EPS)
                fma4(acc, __ldg(val + e), ldg4(frame_row<const float>(x, __ldg(col + e)) + 4 * gl));
            part[slot][gl] = acc;
            __syncthreads();
            for (int h = EPS / 2; h > 0; h >>= 1) {
                if (slot < h) {
                    const float4 o = part[slot + h][gl];
                    float4 v = part[slot][gl];
                    v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                    part[slot][gl] = v;
                }
                __syncthreads();
            }
            const float* sv = reinterpret_cast<const float*>(&part[0][0]);
            emit(row, part[0][gl], threadIdx.x < G, threadIdx.x, blockDim.x, sv);
            __syncthreads();
        }
        __syncthreads();
    }
}

template <int F, int H, int MODE>
int hub_rows_t(int32_t n, const int32_t* rp, const int32_t* col, const float* val, dgnn_frame x, const float* w,
               dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st) {
    int64_t blocks = cdiv(n, 256);
    blocks = blocks > 4 * num_sms() ? 4 * num_sms() : (blocks < 1 ? 1 : blocks);
    ::dgnn::note_launch();
    hub_rows_kernel<F, H, MODE><<<(unsigned)blocks, 256, 0, st>>>(n, rp, col, val, x, w, s_out, r_out);
    return launch_status("hub_rows");
}

// K3 for the 4-wide first layer (s = s1 rows, no aggregation): HP / 4 lanes
// per row, each computing one float4 of q = s W in the same fmaf order as
// gcn_fwd_kernel (bitwise equal) and storing it coalesced (a row-per-lane
// layout would scatter 32 rows per store instruction).
template <int HP, bool SKIP>
__global__ void __launch_bounds__(256) gcn_fwd_narrow_kernel(int32_t n, dgnn_frame x, const float* __restrict__ w,
                                                             dgnn_frame s_out, dgnn_frame r_out) {
    constexpr int LPR = HP / 4 >= 32 ? 32 : HP / 4, RPW = 32 / LPR, QV = HP / (4 * LPR);
    __shared__ float4 wsm4[HP];   // 4 x HP
    for (int i = threadIdx.x; i < HP; i += blockDim.x) wsm4[i] = reinterpret_cast<const float4*>(w)[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, sub = lane / LPR, gl = lane % LPR;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = warp * RPW + sub; row < n; row += nwarps * RPW) {
        const float4 sv = ldg4(frame_row<const float>(x, row));
        float* rr = frame_row<float>(r_out, row);
#pragma unroll
        for (int i = 0; i < QV; ++i) {
            const int c4 = gl + LPR * i;
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) fma4(q, comp(sv, kk), wsm4[kk * (HP / 4) + c4]);
            st4(rr + (SKIP ? 4 : 0) + 4 * c4, relu4(q));
        }
        if (gl == 0) {
            if (s_out.ptr) st4(frame_row<float>(s_out, row), sv);
            if (SKIP) st4(rr, relu4(sv));
        }
    }
}

// K3: s = Ahat x (or x), q = s W, r = relu([s, q]) | relu(q)
template <int FP, int HP, bool SKIP, bool AGG>
__global__ void __launch_bounds__(256) gcn_fwd_kernel(int32_t n, const int32_t* __restrict__ rp,
                                                      const int32_t* __restrict__ col,
                                                      const float* __restrict__ val, dgnn_frame x,
                                                      const float* __restrict__ w, dgnn_frame s_out,
                                                      dgnn_frame r_out) {
    constexpr int G = FP / 4, RW = 32 / G;
    constexpr int QLANES = HP >= FP ? G : HP / 4;   // lanes that own q columns
    constexpr int QV = HP >= FP ? HP / FP : 1;      // float4 q chunks per owning lane
    extern __shared__ float4 wsm4[];
    for (int i = threadIdx.x; i < FP * HP / 4; i += blockDim.x) wsm4[i] = reinterpret_cast<const float4*>(w)[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * RW; base < n; base += nwarps * RW) {
        const int64_t row = base + sub;
        const bool valid = row < n;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
            if constexpr (AGG) s = gather_row(row, rp, col, val, x, gl);
            else s = ldg4(frame_row<const float>(x, row) + 4 * gl);
        }
        float4 q[QV];
#pragma unroll
        for (int i = 0; i < QV; ++i) q[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k4 = 0; k4 < G; ++k4) {
            const int src = sub * G + k4;
            float4 sk;
            sk.x = __shfl_sync(0xffffffffu, s.x, src);
            sk.y = __shfl_sync(0xffffffffu, s.y, src);
            sk.z = __shfl_sync(0xffffffffu, s.z, src);
            sk.w = __shfl_sync(0xffffffffu, s.w, src);
            if (gl < QLANES) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const float sv = comp(sk, kk);
                    const float4* wr = wsm4 + (4 * k4 + kk) * (HP / 4);
#pragma unroll
                    for (int i = 0; i < QV; ++i) fma4(q[i], sv, wr[gl + G * i]);
                }
            }
        }
        if (valid) {
            if (s_out.ptr) st4(frame_row<float>(s_out, row) + 4 * gl, s);
            float* rr = frame_row<float>(r_out, row);
            if constexpr (SKIP) {
                st4(rr + 4 * gl, relu4(s));
                if (gl < QLANES) {
#pragma unroll
                    for (int i = 0; i < QV; ++i) st4(rr + FP + 4 * (gl + G * i), relu4(q[i]));
                }
            } else {
                if (gl < QLANES) {
#pragma unroll
                    for (int i = 0; i < QV; ++i) st4(rr + 4 * (gl + G * i), relu4(q[i]));
                }
            }
        }
    }
}

// K4 row part: dpre = dr (.) [r > 0]; ds = [dpre_s] + dq W^T
template <int FP, int HP, bool SKIP>
__global__ void __launch_bounds__(256) gcn_bwd_rows_kernel(int32_t n, dgnn_frame dr, dgnn_frame r,
                                                           const float* __restrict__ w, dgnn_frame ds) {
    constexpr int G = FP / 4, RW = 32 / G;
    constexpr int QLANES = HP >= FP ? G : HP / 4;
    constexpr int QV = HP >= FP ? HP / FP : 1;
    constexpr int OFF = SKIP ? FP : 0;
    extern __shared__ float4 wt4[];  // W^T: [HP][FP]
    float* wt = reinterpret_cast<float*>(wt4);
    for (int i = threadIdx.x; i < FP * HP; i += blockDim.x) {
        const int k = i / HP, j = i % HP;
        wt[j * FP + k] = w[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * RW; base < n; base += nwarps * RW) {
        const int64_t row = base + sub;
        const bool valid = row < n;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 dq[QV];
#pragma unroll
        for (int i = 0; i < QV; ++i) dq[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
            const float* drr = frame_row<const float>(dr, row);
            const float* rr = frame_row<const float>(r, row);
            if constexpr (SKIP) {
                const float4 g = ldg4(drr + 4 * gl), m = ldg4(rr + 4 * gl);
                acc = make_float4(m.x > 0.f ? g.x : 0.f, m.y > 0.f ? g.y : 0.f, m.z > 0.f ? g.z : 0.f,
                                  m.w > 0.f ? g.w : 0.f);
            }
            if (gl < QLANES) {
#pragma unroll
                for (int i = 0; i < QV; ++i) {
                    const int c = OFF + 4 * (gl + G * i);
                    const float4 g = ldg4(drr + c), m = ldg4(rr + c);
                    dq[i] = make_float4(m.x > 0.f ? g.x : 0.f, m.y > 0.f ? g.y : 0.f, m.z > 0.f ? g.z : 0.f,
                                        m.w > 0.f ? g.w : 0.f);
                }
            }
        }
#pragma unroll
        for (int src = 0; src < QLANES; ++src) {
#pragma unroll
            for (int i = 0; i < QV; ++i) {
                float4 d;
                const int sl = sub * G + src;
                d.x = __shfl_sync(0xffffffffu, dq[i].x, sl);
                d.y = __shfl_sync(0xffffffffu, dq[i].y, sl);
                d.z = __shfl_sync(0xffffffffu, dq[i].z, sl);
                d.w = __shfl_sync(0xffffffffu, dq[i].w, sl);
                const int j0 = 4 * (src + G * i);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) fma4(acc, comp(d, jj), wt4[((j0 + jj) * FP) / 4 + gl]);
            }
        }
        if (valid) st4(frame_row<float>(ds, row) + 4 * gl, acc);
    }
}

// tcgen05 instance of K3 (gcn_tc.cu); -1 when the shape has none
int gcn_fwd_tc(int fp, int hp, bool skip, bool agg, int32_t n, const int32_t* rp, const int32_t* col,
               const float* val, dgnn_frame x, const float* w, dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st);
int gcn_bwd_tc(int fp, int hp, bool skip, int32_t n, dgnn_frame dr, dgnn_frame r, const float* w, dgnn_frame ds,
               cudaStream_t st);


}  // namespace dgnn

using namespace dgnn;

namespace {

template <int F>
int spmm_f32_t(int32_t n, const int32_t* rp, const int32_t* col, const float* val, dgnn_frame x,
               dgnn_frame out, cudaStream_t st) {
    constexpr int RW = 32 / (F / 4);
    int64_t blocks = cdiv(cdiv(n, RW), 8);
    blocks = blocks < 1 ? 1 : (blocks > 32 * num_sms() ? 32 * num_sms() : blocks);
    ::dgnn::note_launch();
    spmm_f32_kernel<F><<<(unsigned)blocks, 256, 0, st>>>(n, rp, col, val, x, out);
    const int rc = launch_status("spmm_f32");
    if (rc) return rc;
    return hub_rows_t<F, 4, 0>(n, rp, col, val, x, nullptr, dgnn_frame{}, out, st);
}

template <int FP, int HP, bool SKIP, bool AGG>
int gcn_fwd_t(int32_t n, const int32_t* rp, const int32_t* col, const float* val, dgnn_frame x, const float* w,
              dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st) {
    if constexpr (FP == 4 && !AGG) {
        constexpr int LPR = HP / 4 >= 32 ? 32 : HP / 4, RPW = 32 / LPR;
        int64_t blocks = cdiv(cdiv(n, RPW), 8);
        blocks = blocks < 1 ? 1 : (blocks > 16 * num_sms() ? 16 * num_sms() : blocks);
        ::dgnn::note_launch();
        gcn_fwd_narrow_kernel<HP, SKIP><<<(unsigned)blocks, 256, 0, st>>>(n, x, w, s_out, r_out);
        return launch_status("gcn_forward (narrow)");
    }
    constexpr int RW = 32 / (FP / 4);
    const size_t smem = (size_t)FP * HP * sizeof(float);
    auto k = gcn_fwd_kernel<FP, HP, SKIP, AGG>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int64_t blocks = cdiv(cdiv(n, RW), 8);
    blocks = blocks < 1 ? 1 : (blocks > 16 * num_sms() ? 16 * num_sms() : blocks);
    ::dgnn::note_launch();
    k<<<(unsigned)blocks, 256, smem, st>>>(n, rp, col, val, x, w, s_out, r_out);
    return launch_status("gcn_forward");
}

template <int FP, int HP, bool SKIP>
int gcn_bwd_t(int32_t n, dgnn_frame dr, dgnn_frame r, const float* w, dgnn_frame ds, cudaStream_t st) {
    constexpr int RW = 32 / (FP / 4);
    const size_t smem = (size_t)FP * HP * sizeof(float);
    auto k = gcn_bwd_rows_kernel<FP, HP, SKIP>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int64_t blocks = cdiv(cdiv(n, RW), 8);
    blocks = blocks < 1 ? 1 : (blocks > 16 * num_sms() ? 16 * num_sms() : blocks);
    ::dgnn::note_launch();
    k<<<(unsigned)blocks, 256, smem, st>>>(n, dr, r, w, ds);
    return launch_status("gcn_backward_rows");
}

template <int FP, bool SKIP, bool AGG>
int gcn_fwd_hp(int32_t hp, int32_t n, const int32_t* rp, const int32_t* col, const float* val, dgnn_frame x,
               const float* w, dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st) {
    switch (hp) {
        case 16: return gcn_fwd_t<FP, 16, SKIP, AGG>(n, rp, col, val, x, w, s_out, r_out, st);
        case 32: return gcn_fwd_t<FP, 32, SKIP, AGG>(n, rp, col, val, x, w, s_out, r_out, st);
        case 64: return gcn_fwd_t<FP, 64, SKIP, AGG>(n, rp, col, val, x, w, s_out, r_out, st);
        case 128: return gcn_fwd_t<FP, 128, SKIP, AGG>(n, rp, col, val, x, w, s_out, r_out, st);
    }
    set_error("gcn_forward: unsupported hp %d", hp);
    return DGNN_EUNSUPPORTED;
}

template <bool SKIP, bool AGG>
int gcn_fwd_fp(int32_t fp, int32_t hp, int32_t n, const int32_t* rp, const int32_t* col, const float* val,
               dgnn_frame x, const float* w, dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st) {
    switch (fp) {
        case 4:
            if (AGG) break;
            return gcn_fwd_hp<4, SKIP, false>(hp, n, rp, col, val, x, w, s_out, r_out, st);
        case 16: return gcn_fwd_hp<16, SKIP, AGG>(hp, n, rp, col, val, x, w, s_out, r_out, st);
        case 32: return gcn_fwd_hp<32, SKIP, AGG>(hp, n, rp, col, val, x, w, s_out, r_out, st);
        case 64: return gcn_fwd_hp<64, SKIP, AGG>(hp, n, rp, col, val, x, w, s_out, r_out, st);
        case 128: return gcn_fwd_hp<128, SKIP, AGG>(hp, n, rp, col, val, x, w, s_out, r_out, st);
    }
    set_error("gcn_forward: unsupported fp %d (aggregation %d)", fp, (int)AGG);
    return DGNN_EUNSUPPORTED;
}

template <int FP, bool SKIP>
int gcn_bwd_hp(int32_t hp, int32_t n, dgnn_frame dr, dgnn_frame r, const float* w, dgnn_frame ds, cudaStream_t st) {
    switch (hp) {
        case 16: return gcn_bwd_t<FP, 16, SKIP>(n, dr, r, w, ds, st);
        case 32: return gcn_bwd_t<FP, 32, SKIP>(n, dr, r, w, ds, st);
        case 64: return gcn_bwd_t<FP, 64, SKIP>(n, dr, r, w, ds, st);
        case 128: return gcn_bwd_t<FP, 128, SKIP>(n, dr, r, w, ds, st);
    }
    set_error("gcn_backward_rows: unsupported hp %d", hp);
    return DGNN_EUNSUPPORTED;
}

template <bool SKIP>
int gcn_bwd_fp(int32_t fp, int32_t hp, int32_t n, dgnn_frame dr, dgnn_frame r, const float* w, dgnn_frame ds,
               cudaStream_t st) {
    switch (fp) {
        case 4: return gcn_bwd_hp<4, SKIP>(hp, n, dr, r, w, ds, st);
        case 16: return gcn_bwd_hp<16, SKIP>(hp, n, dr, r, w, ds, st);
        case 32: return gcn_bwd_hp<32, SKIP>(hp, n, dr, r, w, ds, st);
        case 64: return gcn_bwd_hp<64, SKIP>(hp, n, dr, r, w, ds, st);
        case 128: return gcn_bwd_hp<128, SKIP>(hp, n, dr, r, w, ds, st);
    }
    set_error("gcn_backward_rows: unsupported fp %d", fp);
    return DGNN_EUNSUPPORTED;
}

}  // namespace

// hub rows of the fused GCN forward (both instances)
template <int F>
int gcn_hub_rows_h(int hp, bool skip, int32_t n, const int32_t* rp, const int32_t* col, const float* val,
                   dgnn_frame x, const float* w, dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st) {
    switch (hp) {
#define HUB_H(H)                                                                                   \
    case H:                                                                                        \
        return skip ? hub_rows_t<F, H, 1>(n, rp, col, val, x, w, s_out, r_out, st)                \
                    : hub_rows_t<F, H, 2>(n, rp, col, val, x, w, s_out, r_out, st);
        HUB_H(16) HUB_H(32) HUB_H(64) HUB_H(128)
#undef HUB_H
    }
    set_error("gcn_forward: unsupported hp %d", hp);
    return DGNN_EUNSUPPORTED;
}

int gcn_hub_rows(int fp, int hp, bool skip, int32_t n, const int32_t* rp, const int32_t* col, const float* val,
                 dgnn_frame x, const float* w, dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st) {
    switch (fp) {
        case 16: return gcn_hub_rows_h<16>(hp, skip, n, rp, col, val, x, w, s_out, r_out, st);
        case 32: return gcn_hub_rows_h<32>(hp, skip, n, rp, col, val, x, w, s_out, r_out, st);
        case 64: return gcn_hub_rows_h<64>(hp, skip, n, rp, col, val, x, w, s_out, r_out, st);
        case 128: return gcn_hub_rows_h<128>(hp, skip, n, rp, col, val, x, w, s_out, r_out, st);
    }
    set_error("gcn_forward: unsupported fp %d", fp);
    return DGNN_EUNSUPPORTED;
}

extern "C" {

// K3 engine selection: tcgen05 instance where one exists (default) or the
// SIMT kernel (A/B and strict-tolerance tests); dgnn_set_gcn_tensor_cores.
static int dgnn_gcn_tensor_cores = 1;

void dgnn_set_gcn_tensor_cores(int on) { dgnn_gcn_tensor_cores = on != 0; }

}  // extern "C"

namespace dgnn {
int gcn_tensor_cores_on() { return dgnn_gcn_tensor_cores; }
}  // namespace dgnn

extern "C" {

int dgnn_spmm_f32(int32_t n, const int32_t* rowptr, const int32_t* col, const float* val, dgnn_frame x,
                  int32_t f, dgnn_frame out, void* stream) {
    DGNN_CHECK_ARG(n >= 0, "spmm_f32: negative size");
    if (n == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (f) {
        case 4: return spmm_f32_t<4>(n, rowptr, col, val, x, out, st);
        case 16: return spmm_f32_t<16>(n, rowptr, col, val, x, out, st);
        case 32: return spmm_f32_t<32>(n, rowptr, col, val, x, out, st);
        case 64: return spmm_f32_t<64>(n, rowptr, col, val, x, out, st);
        case 128: return spmm_f32_t<128>(n, rowptr, col, val, x, out, st);
    }
    set_error("spmm_f32: unsupported width %d", f);
    return DGNN_EUNSUPPORTED;
}

int dgnn_gcn_forward(int32_t n, const int32_t* rowptr, const int32_t* col, const float* val, dgnn_frame x,
                     int32_t fp, const float* w, int32_t hp, int skip, dgnn_frame s_out, dgnn_frame r_out,
                     void* stream) {
    DGNN_CHECK_ARG(n >= 0, "gcn_forward: negative size");
    if (n == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    const bool agg = rowptr != nullptr;
    int rc = -1;
    if (dgnn_gcn_tensor_cores) rc = gcn_fwd_tc(fp, hp, skip != 0, agg, n, rowptr, col, val, x, w, s_out, r_out, st);
    if (rc < 0) {
        if (skip)
            rc = agg ? gcn_fwd_fp<true, true>(fp, hp, n, rowptr, col, val, x, w, s_out, r_out, st)
                     : gcn_fwd_fp<true, false>(fp, hp, n, rowptr, col, val, x, w, s_out, r_out, st);
        else
            rc = agg ? gcn_fwd_fp<false, true>(fp, hp, n, rowptr, col, val, x, w, s_out, r_out, st)
                     : gcn_fwd_fp<false, false>(fp, hp, n, rowptr, col, val, x, w, s_out, r_out, st);
    }
    if (rc || !agg) return rc;
    return gcn_hub_rows(fp, hp, skip != 0, n, rowptr, col, val, x, w, s_out, r_out, st);
}

int dgnn_gcn_backward_rows(int32_t n, dgnn_frame dr, dgnn_frame r, int32_t fp, const float* w, int32_t hp,
                           int skip, dgnn_frame ds, void* stream) {
    DGNN_CHECK_ARG(n >= 0, "gcn_backward_rows: negative size");
    if (n == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    if (dgnn_gcn_tensor_cores) {
        const int rc = gcn_bwd_tc(fp, hp, skip != 0, n, dr, r, w, ds, st);
        if (rc >= 0) return rc;
    }
    return skip ? gcn_bwd_fp<true>(fp, hp, n, dr, r, w, ds, st) : gcn_bwd_fp<false>(fp, hp, n, dr, r, w, ds, st);
}

}  // extern "C"
