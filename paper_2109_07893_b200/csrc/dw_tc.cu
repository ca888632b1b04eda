// LSTM weight gradients on tcgen05 (the x^T dz, h^T dz, sum dz products of
// training.py:422-424, over every vertex row of every step of a block):
//
//   S[j][k] = sum_r dz[r][j] * xcat[r][k],   xcat[r] = [x_t[v] | h_{t-1}[v]],
//   db[j]   = sum_r dz[r][j],                r = t * NP + v.
//
// Both operands are staged MN-major straight from their row-major HBM
// layout (a 128-byte row segment of 32 columns is one swizzle-atom row), so
// nothing is transposed: A = dz^T (M = 4*HP gate columns, one or two M=128
// tiles), B = xcat^T (N = kx + HP rounded to 16), K = rows.  3xTF32 split as in
// lstm_tc.cu.  One persistent CTA per SM owns a contiguous row range.
//
// tcgen05 fp32 accumulation truncates, so a TMEM accumulator only lives for
// DW_PERIOD rows; then it is promoted (fp32, round-to-nearest) into the CTA's
// own slot in global memory (L2 resident) and restarted.  The CTA slots are
// reduced in fp64 in fixed order by a second kernel: deterministic.
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

constexpr int DW_ROWS = 16;      // reduction rows per stage = two 8-row K groups
constexpr int DW_PERIOD = 512;   // rows per TMEM accumulation period
constexpr int DW_STAGES = 3;

struct DwShape {
    int M, mtile, mt, N, atoms_a, atoms_b, a_half, b_half, stage, tmem_cols;
};

__host__ __device__ inline DwShape dw_shape(int hp, int kx) {
    DwShape s;
    s.M = 4 * hp;
    s.mtile = s.M < 128 ? s.M : 128;
    s.mt = s.M / s.mtile;
    s.N = (kx + hp + 31) / 32 * 32;   // MN atoms are 32 elements wide
    s.atoms_a = s.M / 32;
    s.atoms_b = s.N / 32;
    s.a_half = 4 * s.atoms_a * 512;   // hi (or lo) part: 4 K groups (of 4 rows) x atoms x 512 B
    s.b_half = 4 * s.atoms_b * 512;
    s.stage = 2 * s.a_half + 2 * s.b_half;
    const int cols = s.mt * s.N;
    s.tmem_cols = cols <= 32 ? 32 : (cols <= 64 ? 64 : (cols <= 128 ? 128 : (cols <= 256 ? 256 : 512)));
    return s;
}

inline size_t dw_smem_bytes(const DwShape& s) { return (size_t)DW_STAGES * s.stage + 1024 + 128; }

// MN-major tf32 operands must use SWIZZLE_128B_BASE32B (CUTLASS
// Layout_MN_SW128_32B_Atom): a 512-byte atom holds 4 K rows x 32 MN elements
// (128 B per row), and 32-byte granule c of row r sits at granule c ^ r.
// Byte offset of (row r in stage, column c) inside one operand half laid out
// [K group (4 rows)][MN atom][512 B]; c must be a multiple of 4.
constexpr uint32_t kSW128B32 = 1;
__device__ __forceinline__ uint32_t mn_off(int r, int c, int atoms) {
    const int g = r >> 2, r4 = r & 3, j = c >> 5, e = c & 31;
    return (uint32_t)((g * atoms + j) * 512 + r4 * 128 + ((((e >> 3) ^ r4) & 3) << 5) + ((e & 7) << 2));
}

template <int HP>
__global__ void __launch_bounds__(256, 1) lstm_dw_tc_kernel(int64_t rows, int64_t np, int kx,
                                                            const float* __restrict__ x, int64_t ldx,
                                                            const float* __restrict__ y,
                                                            const float* __restrict__ h0,
                                                            const float* __restrict__ dz,
                                                            float* __restrict__ slots, double* __restrict__ dbs) {
    constexpr int M = 4 * HP;
    constexpr int AV = (DW_ROWS * M / 4) / 256;      // A float4 items per thread per stage
    const DwShape S = dw_shape(HP, kx);
    const int K = kx + HP;
    const int BVEC = DW_ROWS * S.N / 4;              // B float4 items per stage
    constexpr int BMAX = (DW_ROWS * 256 / 4 + 255) / 256;

    extern __shared__ uint8_t dw_smem_raw[];
    const uint32_t raw = smem_u32(dw_smem_raw);
    uint8_t* base = dw_smem_raw + ((1024 - (raw & 1023)) & 1023);
    const uint32_t sb = smem_u32(base);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + DW_STAGES * S.stage);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + DW_STAGES);
    const int tid = threadIdx.x;
    if (tid < 32) tmem_alloc(tslot, S.tmem_cols);
    if (tid == 32) {
        for (int i = 0; i < DW_STAGES; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;

    // contiguous row range of this CTA (multiple of 16)
    const int64_t per = cdiv(cdiv(rows, gridDim.x), DW_ROWS) * DW_ROWS;
    const int64_t r_begin = blockIdx.x * per;
    const int64_t r_end = min(rows, r_begin + per);
    const int nst = r_end > r_begin ? (int)cdiv(r_end - r_begin, DW_ROWS) : 0;
    const int period_st = DW_PERIOD / DW_ROWS;
    float* slot = slots + (size_t)blockIdx.x * M * S.N;

    float4 ca[AV], na[AV], cb[BMAX], nb[BMAX];
    double dbacc[4] = {0.0, 0.0, 0.0, 0.0};
    auto fetch = [&](int st, float4* va, float4* vb) {
        const int64_t r0 = r_begin + (int64_t)st * DW_ROWS;
#pragma unroll
        for (int i = 0; i < AV; ++i) {
            const int idx = tid + 256 * i;
            const int r = idx / (M / 4), c = 4 * (idx % (M / 4));
            const int64_t g = r0 + r;
            va[i] = g < r_end ? __ldg(reinterpret_cast<const float4*>(dz + g * M + c))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < BMAX; ++i) {
            const int idx = tid + 256 * i;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (idx < BVEC) {
                const int r = idx / (S.N / 4), c = 4 * (idx % (S.N / 4));
                const int64_t g = r0 + r;
                if (g < r_end && c < K) {
                    if (c < kx) v = __ldg(reinterpret_cast<const float4*>(x + g * ldx + c));
                    else if (g >= np) v = __ldg(reinterpret_cast<const float4*>(y + (g - np) * HP + (c - kx)));
                    else v = __ldg(reinterpret_cast<const float4*>(h0 + g * HP + (c - kx)));
                }
            }
            vb[i] = v;
        }
    };
    if (nst > 0) fetch(0, ca, cb);

    const int w = tid >> 5, lane = tid & 31, q = w & 3, half = w >> 2;
    for (int st = 0; st < nst; ++st) {
        const int s = st % DW_STAGES;
        if (st + 1 < nst) fetch(st + 1, na, nb);
        if (st >= DW_STAGES) mbar_wait(&bars[s], ((st - DW_STAGES) / DW_STAGES) & 1);
        const uint32_t a_hi = sb + s * S.stage, a_lo = a_hi + S.a_half;
        const uint32_t b_hi = a_lo + S.a_half, b_lo = b_hi + S.b_half;
#pragma unroll
        for (int i = 0; i < AV; ++i) {
            const int idx = tid + 256 * i;
            const int r = idx / (M / 4), c = 4 * (idx % (M / 4));
            float4 hi, lo;
            split4(ca[i], hi, lo);
            const uint32_t o = mn_off(r, c, S.atoms_a);
            sts128(a_hi + o, hi);
            sts128(a_lo + o, lo);
            dbacc[0] += ca[i].x;
            dbacc[1] += ca[i].y;
            dbacc[2] += ca[i].z;
            dbacc[3] += ca[i].w;
        }
#pragma unroll
        for (int i = 0; i < BMAX; ++i) {
            const int idx = tid + 256 * i;
            if (idx < BVEC) {
                const int r = idx / (S.N / 4), c = 4 * (idx % (S.N / 4));
                float4 hi, lo;
                split4(cb[i], hi, lo);
                const uint32_t o = mn_off(r, c, S.atoms_b);
                sts128(b_hi + o, hi);
                sts128(b_lo + o, lo);
            }
        }
        fence_async_smem();
        __syncthreads();
        const bool first = (st % period_st) == 0;
        if (tid == 0) {
            fence_after();
            const uint32_t idesc = idesc_tf32_mn(S.mtile, S.N);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const uint64_t bh = sdesc_mn(b_hi + 2 * kk * S.atoms_b * 512, 512, S.atoms_b * 512, kSW128B32);
                const uint64_t bl = sdesc_mn(b_lo + 2 * kk * S.atoms_b * 512, 512, S.atoms_b * 512, kSW128B32);
                for (int m = 0; m < S.mt; ++m) {
                    const uint32_t aoff = (2 * kk * S.atoms_a + m * (S.mtile / 32)) * 512;
                    const uint64_t ah = sdesc_mn(a_hi + aoff, 512, S.atoms_a * 512, kSW128B32);
                    const uint64_t al = sdesc_mn(a_lo + aoff, 512, S.atoms_a * 512, kSW128B32);
                    const uint32_t d = tmem + m * S.N;
                    mma_tf32(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                    mma_tf32(d, ah, bl, idesc, 1u);
                    mma_tf32(d, al, bh, idesc, 1u);
                }
            }
            commit(&bars[s]);
        }
        const bool end_of_period = ((st + 1) % period_st) == 0 || st + 1 == nst;
        if (end_of_period) {
            // promotion: TMEM period sum -> fp32 slot (round to nearest)
            mbar_wait(&bars[s], (st / DW_STAGES) & 1);
            fence_after();
            const bool first_period = st < period_st;
            for (int m = 0; m < S.mt; ++m) {
                const int j = m * S.mtile + 32 * q + lane;
                for (int c0 = half * 8; c0 < S.N; c0 += 16) {
                    float v[8];
                    tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + m * S.N + c0, v);
                    tmem_wait_ld();
                    if (32 * q + lane < S.mtile) {
                        float4* o = reinterpret_cast<float4*>(slot + (size_t)j * S.N + c0);
                        float4 a = make_float4(v[0], v[1], v[2], v[3]), b = make_float4(v[4], v[5], v[6], v[7]);
                        if (!first_period) {
                            const float4 p0 = o[0], p1 = o[1];
                            a.x += p0.x; a.y += p0.y; a.z += p0.z; a.w += p0.w;
                            b.x += p1.x; b.y += p1.y; b.z += p1.z; b.w += p1.w;
                        }
                        o[0] = a;
                        o[1] = b;
                    }
                }
            }
            fence_before();
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < AV; ++i) ca[i] = na[i];
#pragma unroll
        for (int i = 0; i < BMAX; ++i) cb[i] = nb[i];
    }
    // db partial: threads sharing a column group combine in fixed order
    __shared__ double dbred[256][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) dbred[tid][j] = dbacc[j];
    __syncthreads();
    if (tid < M / 4) {
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int t = tid; t < 256; t += M / 4)
            for (int j = 0; j < 4; ++j) s4[j] += dbred[t][j];
        for (int j = 0; j < 4; ++j) dbs[(size_t)blockIdx.x * M + 4 * tid + j] = s4[j];
    }
    if (nst == 0) {   // empty range: publish zeros
        for (int i = tid; i < M * S.N; i += 256) slot[i] = 0.f;
    }
    fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(tmem, S.tmem_cols);
}

// gw[k][j] += sum_cta slot[cta][j][k] ; gb[j] += sum_cta dbs[cta][j]   (fp64, fixed order)
__global__ void dw_reduce_kernel(int nct, int M, int N, int K, const float* __restrict__ slots,
                                 const double* __restrict__ dbs, double* __restrict__ gw, int64_t ldg,
                                 double* __restrict__ gb) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < (int64_t)M * K) {
        const int k = (int)(i / M), j = (int)(i % M);
        double s = 0.0;
        for (int c = 0; c < nct; ++c) s += (double)slots[((size_t)c * M + j) * N + k];
        gw[(int64_t)k * ldg + j] += s;
    } else if (i < (int64_t)M * K + M && gb) {
        const int j = (int)(i - (int64_t)M * K);
        double s = 0.0;
        for (int c = 0; c < nct; ++c) s += dbs[(size_t)c * M + j];
        gb[j] += s;
    }
}

template <int HP>
int lstm_dw_tc_t(int64_t rows, int64_t np, int kx, const float* x, int64_t ldx, const float* y, const float* h0,
                 const float* dz, double* gw, double* gb, void* ws, size_t ws_bytes, cudaStream_t st) {
    const DwShape S = dw_shape(HP, kx);
    if (S.mt * S.N > 512 || S.N > 256) {
        set_error("lstm_weight_grad_tc: kx + hp = %d too wide", kx + HP);
        return DGNN_EUNSUPPORTED;
    }
    const int grid = kSMs;
    const size_t need = (size_t)grid * S.M * S.N * sizeof(float) + (size_t)grid * S.M * sizeof(double);
    if (ws_bytes < need) {
        set_error("lstm_weight_grad_tc: workspace too small");
        return DGNN_EWORKSPACE;
    }
    float* slots = reinterpret_cast<float*>(ws);
    double* dbs = reinterpret_cast<double*>(slots + (size_t)grid * S.M * S.N);
    auto k = lstm_dw_tc_kernel<HP>;
    const size_t smem = dw_smem_bytes(S);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch();
    k<<<grid, 256, smem, st>>>(rows, np, kx, x, ldx, y, h0, dz, slots, dbs);
    const int K = kx + HP;
    const int64_t tot = (int64_t)S.M * K + S.M;
    note_launch();
    dw_reduce_kernel<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(grid, S.M, S.N, K, slots, dbs, gw, S.M, gb);
    return launch_status("lstm_weight_grad_tc");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

size_t dgnn_lstm_weight_grad_tc_workspace(int32_t kx, int32_t hp) {
    const DwShape S = dw_shape(hp, kx);
    return (size_t)kSMs * S.M * S.N * sizeof(float) + (size_t)kSMs * S.M * sizeof(double) + 256;
}

int dgnn_lstm_weight_grad_tc(int64_t rows, int64_t np, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                             const float* h_out, const float* h0, const float* dz, double* gwcat, double* gb,
                             void* workspace, size_t workspace_bytes, void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && np > 0 && kx % 4 == 0 && ldx % 4 == 0, "lstm_weight_grad_tc: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 32: return lstm_dw_tc_t<32>(rows, np, kx, x, ldx, h_out, h0, dz, gwcat, gb, workspace, workspace_bytes, st);
        case 64: return lstm_dw_tc_t<64>(rows, np, kx, x, ldx, h_out, h0, dz, gwcat, gb, workspace, workspace_bytes, st);
    }
    set_error("lstm_weight_grad_tc: unsupported hp %d (M = 4hp must be >= 128; use dgnn_gemm_tn)", hp);
    return DGNN_EUNSUPPORTED;
}

}  // extern "C"
