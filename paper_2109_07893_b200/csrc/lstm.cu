// Temporal stage (K5/K6): one LSTM step over a vertex chunk, the gate GEMM
// fused with the cell update, and the reverse step fused with the
// gate-gradient prologue.  Reference: training.py:370-427, models.py:215-239.
//
// SIMT fp32 register-tiled version: a CTA owns BM vertex rows and all 4*HP
// gate columns, so every thread ends the GEMM holding the four gates of its
// (row, unit) pairs and applies the cell update in registers; nothing but
// h, c (and the gate cache when the backward needs it) goes back to HBM.
#include "common.cuh"

namespace dgnn {

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }

// ---------------------------------------------------------------------------
// forward step: z = [x | h_prev] W + b ; gates ; c, h

template <int HP>
struct FwdCfg {
    static constexpr int UG = HP / 2;        // unit pairs across the CTA
    static constexpr int RG = 256 / UG;      // row groups
    static constexpr int RPT = 8;            // rows per thread
    static constexpr int BM = RG * RPT;      // rows per CTA
    static constexpr int BK = 16;
    static constexpr int NC = 4 * HP;
};

template <int HP>
__global__ void __launch_bounds__(256) lstm_fwd_kernel(int64_t rows, int kx, const float* __restrict__ x,
                                                       int64_t ldx, const float* __restrict__ hprev,
                                                       const float* __restrict__ cprev,
                                                       const float* __restrict__ wcat,
                                                       const float* __restrict__ bias, float* __restrict__ hout,
                                                       float* __restrict__ cout, float* __restrict__ gates) {
    using C = FwdCfg<HP>;
    __shared__ __align__(16) float As[C::BK][C::BM];
    __shared__ __align__(16) float Bs[C::BK][C::NC];
    const int tid = threadIdx.x, ug = tid % C::UG, rg = tid / C::UG;
    const int64_t row0 = blockIdx.x * (int64_t)C::BM;
    const int K = kx + HP;
    float acc[C::RPT][8];
#pragma unroll
    for (int i = 0; i < C::RPT; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    for (int k0 = 0; k0 < K; k0 += C::BK) {
        for (int i = tid; i < C::BM * (C::BK / 4); i += 256) {
            const int r = i / (C::BK / 4), c4 = i % (C::BK / 4);
            const int k = k0 + 4 * c4;
            const int64_t g = row0 + r;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (g < rows && k < K) v = k < kx ? ld4(x + g * ldx + k) : ld4(hprev + g * HP + (k - kx));
            As[4 * c4 + 0][r] = v.x;
            As[4 * c4 + 1][r] = v.y;
            As[4 * c4 + 2][r] = v.z;
            As[4 * c4 + 3][r] = v.w;
        }
        for (int i = tid; i < C::BK * (C::NC / 4); i += 256) {
            const int kk = i / (C::NC / 4), c4 = i % (C::NC / 4);
            const int k = k0 + kk;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k < K) v = ld4(wcat + (int64_t)k * C::NC + 4 * c4);
            *reinterpret_cast<float4*>(&Bs[kk][4 * c4]) = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < C::BK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][rg * C::RPT]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][rg * C::RPT + 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            float b[8];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const float2 bv = *reinterpret_cast<const float2*>(&Bs[kk][g * HP + 2 * ug]);
                b[2 * g] = bv.x;
                b[2 * g + 1] = bv.y;
            }
#pragma unroll
            for (int i = 0; i < C::RPT; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }

    const int u0 = 2 * ug;
    float bz[8];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        bz[2 * g] = bias[g * HP + u0];
        bz[2 * g + 1] = bias[g * HP + u0 + 1];
    }
#pragma unroll
    for (int i = 0; i < C::RPT; ++i) {
        const int64_t g = row0 + rg * C::RPT + i;
        if (g >= rows) continue;
        const float2 cp = ld2(cprev + tb_off(g, u0, HP, rows));
        float hv[2], cv[2], gi[2], gf[2], go[2], gg[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            gi[j] = act_sigmoid(acc[i][0 + j] + bz[0 + j]);
            gf[j] = act_sigmoid(acc[i][2 + j] + bz[2 + j]);
            go[j] = act_sigmoid(acc[i][4 + j] + bz[4 + j]);
            gg[j] = act_tanh(acc[i][6 + j] + bz[6 + j]);
            const float c_old = j == 0 ? cp.x : cp.y;
            cv[j] = gf[j] * c_old + gi[j] * gg[j];
            hv[j] = go[j] * act_tanh(cv[j]);
        }
        st2(hout + g * HP + u0, hv[0], hv[1]);
        st2(cout + tb_off(g, u0, HP, rows), cv[0], cv[1]);
        if (gates) {
            st2(gates + tb_off(g, 0 * HP + u0, C::NC, rows), gi[0], gi[1]);
            st2(gates + tb_off(g, 1 * HP + u0, C::NC, rows), gf[0], gf[1]);
            st2(gates + tb_off(g, 2 * HP + u0, C::NC, rows), go[0], go[1]);
            st2(gates + tb_off(g, 3 * HP + u0, C::NC, rows), gg[0], gg[1]);
        }
    }
}

// ---------------------------------------------------------------------------
// backward step: dz (pointwise) then [dx | dh_carry] = dz W^T

template <int HP>
struct BwdCfg {
    static constexpr int NC = 4 * HP;
    static constexpr int BM = HP >= 128 ? 32 : 64;
    static constexpr int TRG = BM / 4;        // row groups of 4 rows
    static constexpr int TKG = 256 / TRG;     // column groups of 4 columns
    static constexpr int KC = 4 * TKG;        // output columns per pass
    static constexpr int BJ = 32;             // reduction chunk
    static constexpr size_t smem = (size_t)(NC * BM + BJ * KC) * sizeof(float);
};

template <int HP>
__global__ void __launch_bounds__(256) lstm_bwd_kernel(int64_t rows, int kx, const float* __restrict__ dy,
                                                       const float* __restrict__ dh_in,
                                                       const float* __restrict__ dc_in, const float* gates,
                                                       const float* __restrict__ cprev,
                                                       const float* __restrict__ cnew,
                                                       const float* __restrict__ wcat_t, float* dz,
                                                       float* __restrict__ dx, int64_t lddx,
                                                       float* __restrict__ dh_out, float* __restrict__ dc_out) {
    using C = BwdCfg<HP>;
    extern __shared__ __align__(16) float sm[];
    float* dzs = sm;                    // [NC][BM]
    float* ws = sm + C::NC * C::BM;     // [BJ][KC]
    const int tid = threadIdx.x;
    const int64_t row0 = blockIdx.x * (int64_t)C::BM;

    // phase 1: gate gradients (training.py:405-421)
    for (int idx = tid; idx < C::BM * HP; idx += 256) {
        const int r = idx / HP, u = idx % HP;
        const int64_t g = row0 + r;
        float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
        if (g < rows) {
            const float gi = gates[tb_off(g, u, C::NC, rows)], gf = gates[tb_off(g, HP + u, C::NC, rows)],
                        go = gates[tb_off(g, 2 * HP + u, C::NC, rows)], gg = gates[tb_off(g, 3 * HP + u, C::NC, rows)];
            const int64_t o = tb_off(g, u, HP, rows);
            const float cp = cprev[o], cn = cnew[o];
            const float tc = act_tanh(cn);
            const float dh = (dy ? dy[g * HP + u] : 0.f) + dh_in[g * HP + u];
            const float d_o = dh * tc;
            const float dc = dh * go * (1.f - tc * tc) + dc_in[o];
            const float df = dc * cp, di = dc * gg, dg = dc * gi;
            dc_out[o] = dc * gf;
            z0 = di * gi * (1.f - gi);
            z1 = df * gf * (1.f - gf);
            z2 = d_o * go * (1.f - go);
            z3 = dg * (1.f - gg * gg);
            dz[tb_off(g, u, C::NC, rows)] = z0;
            dz[tb_off(g, HP + u, C::NC, rows)] = z1;
            dz[tb_off(g, 2 * HP + u, C::NC, rows)] = z2;
            dz[tb_off(g, 3 * HP + u, C::NC, rows)] = z3;
        }
        dzs[(0 * HP + u) * C::BM + r] = z0;
        dzs[(1 * HP + u) * C::BM + r] = z1;
        dzs[(2 * HP + u) * C::BM + r] = z2;
        dzs[(3 * HP + u) * C::BM + r] = z3;
    }
    __syncthreads();

    // phase 2: out[r][k] = sum_j dz[r][j] * W[k][j]   (W^T given row-major [NC][K])
    const int K = kx + HP;
    const int tr = tid / C::TKG, tk = tid % C::TKG;
    for (int k0 = 0; k0 < K; k0 += C::KC) {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
        for (int j0 = 0; j0 < C::NC; j0 += C::BJ) {
            for (int i = tid; i < C::BJ * (C::KC / 4); i += 256) {
                const int jj = i / (C::KC / 4), c4 = i % (C::KC / 4);
                const int k = k0 + 4 * c4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (k < K) v = ld4(wcat_t + (int64_t)(j0 + jj) * K + k);
                *reinterpret_cast<float4*>(ws + jj * C::KC + 4 * c4) = v;
            }
            __syncthreads();
#pragma unroll 8
            for (int jj = 0; jj < C::BJ; ++jj) {
                const float4 a = *reinterpret_cast<const float4*>(dzs + (j0 + jj) * C::BM + 4 * tr);
                const float4 b = *reinterpret_cast<const float4*>(ws + jj * C::KC + 4 * tk);
                const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            __syncthreads();
        }
        const int k = k0 + 4 * tk;
        if (k < K) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t g = row0 + 4 * tr + i;
                if (g >= rows) continue;
                const float4 v = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                if (k < kx) *reinterpret_cast<float4*>(dx + g * lddx + k) = v;
                else *reinterpret_cast<float4*>(dh_out + g * HP + (k - kx)) = v;
            }
        }
    }
}

template <int HP>
int lstm_fwd_t(int64_t rows, int kx, const float* x, int64_t ldx, const float* hp_, const float* cp,
               const float* w, const float* b, float* h, float* c, float* gates, cudaStream_t st) {
    const unsigned grid = (unsigned)cdiv(rows, FwdCfg<HP>::BM);
    ::dgnn::note_launch();
    lstm_fwd_kernel<HP><<<grid, 256, 0, st>>>(rows, kx, x, ldx, hp_, cp, w, b, h, c, gates);
    return launch_status("lstm_forward_step");
}

template <int HP>
int lstm_bwd_t(int64_t rows, int kx, const float* dy, const float* dh_in, const float* dc_in, const float* gates,
               const float* cp, const float* cn, const float* wt, float* dz, float* dx, int64_t lddx,
               float* dh_out, float* dc_out, cudaStream_t st) {
    using C = BwdCfg<HP>;
    auto k = lstm_bwd_kernel<HP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
    const unsigned grid = (unsigned)cdiv(rows, C::BM);
    ::dgnn::note_launch();
    k<<<grid, 256, C::smem, st>>>(rows, kx, dy, dh_in, dc_in, gates, cp, cn, wt, dz, dx, lddx, dh_out, dc_out);
    return launch_status("lstm_backward_step");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

int dgnn_lstm_forward_step(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                           const float* h_prev, const float* c_prev, const float* wcat, const float* bias,
                           float* h_out, float* c_out, float* gates, void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && kx >= 0 && kx % 4 == 0 && ldx % 4 == 0, "lstm_forward_step: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 16: return lstm_fwd_t<16>(rows, kx, x, ldx, h_prev, c_prev, wcat, bias, h_out, c_out, gates, st);
        case 32: return lstm_fwd_t<32>(rows, kx, x, ldx, h_prev, c_prev, wcat, bias, h_out, c_out, gates, st);
        case 64: return lstm_fwd_t<64>(rows, kx, x, ldx, h_prev, c_prev, wcat, bias, h_out, c_out, gates, st);
        case 128: return lstm_fwd_t<128>(rows, kx, x, ldx, h_prev, c_prev, wcat, bias, h_out, c_out, gates, st);
    }
    set_error("lstm_forward_step: unsupported hp %d", hp);
    return DGNN_EUNSUPPORTED;
}

int dgnn_lstm_backward_step(int64_t rows, int32_t kx, int32_t hp, const float* dy, const float* dh_in,
                            const float* dc_in, const float* gates, const float* c_prev, const float* c_new,
                            const float* wcat_t, float* dz, float* dx, int64_t lddx, float* dh_out,
                            float* dc_out, void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && kx >= 0 && kx % 4 == 0 && lddx % 4 == 0, "lstm_backward_step: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 16: return lstm_bwd_t<16>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wcat_t, dz, dx, lddx, dh_out, dc_out, st);
        case 32: return lstm_bwd_t<32>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wcat_t, dz, dx, lddx, dh_out, dc_out, st);
        case 64: return lstm_bwd_t<64>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wcat_t, dz, dx, lddx, dh_out, dc_out, st);
        case 128: return lstm_bwd_t<128>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wcat_t, dz, dx, lddx, dh_out, dc_out, st);
    }
    set_error("lstm_backward_step: unsupported hp %d", hp);
    return DGNN_EUNSUPPORTED;
}

}  // extern "C"
