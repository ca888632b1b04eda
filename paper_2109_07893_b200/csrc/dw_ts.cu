// LSTM weight gradients with the dz operand in TMEM (tcgen05 "TS" MMAs):
// the x^T dz, h^T dz, sum dz products of training.py:422-424 over every
// (row, step) of a block -- the same product, promotion and fixed-order
// reduction as dw_tc.cu, with a different operand path.
//
// Why: dw_tc.cu loads both operands global -> registers (two stages ahead)
// and stores the tf32 hi / lo parts into shared memory.  Its probe
// (scripts/dw_probe2.sh) puts the bound on the loads: 4.0 ms at 6M rows,
// 2.26 ms with the loads removed -- two stages of registers are not enough
// bytes in flight, and there is no room for more (80 registers at 21 warps).
// Here:
//   * loader warps stream raw rows with cp.async into a 4-deep landing ring
//     in shared memory (~116 KB in flight per SM, no registers);
//   * A = dz^T goes landing -> registers -> tf32 split -> tcgen05.st into
//     TMEM (lane = gate column, column = row), so the tensor cores read
//     only B = xcat^T from shared memory:  shared-memory traffic per
//     16-row stage ~150 KB (landing in/out, B split stores, B operand
//     reads) against ~230 KB for staging both operands.
//
//   warps 0..7    A converters: warp w owns TMEM lane quarter w % 4 of gate
//                 tile w / 4; thread = gate column j: 16 landed dz values
//                 (conflict-free: 272-byte column-group pitch), split,
//                 16 hi + 16 lo TMEM columns; fp64 db[j];
//   warps 8..15   B converters: landed xcat rows -> split -> SW128_32B
//                 MN-major hi / lo tiles (conflict-free 16-byte stores);
//   warps 16..19  loaders: cp.async (L2 evict-first) of the stage's dz
//                 (64 column groups x 16 rows of the tile-blocked layout)
//                 and xcat rows ([x_t | h_{t-1}]) into the landing slot;
//   warp 20       MMA issuer: per stage 2 K steps x mt tiles x 3 MMAs
//                 D[m] += A(TMEM) . B(smem);
//   warps 21..24  epilogue: promotion of each 512-row accumulation period
//                 into the CTA's fp32 slot (RED, L2 evict-last).
// Results equal dw_tc.cu's up to the accumulation order of the products.
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

namespace dts {
constexpr int ROWS = 16;          // reduction rows per stage = two 8-row K steps
constexpr int PERIOD = 512;       // rows per TMEM accumulation period (as dw_tc.cu)
constexpr int NA = 8, NB = 8, NL = 4;
constexpr int LOAD_WARP = NA + NB, MMA_WARP = LOAD_WARP + NL, NEPI = 4;
constexpr int THREADS = 32 * (MMA_WARP + 1 + NEPI);
constexpr int NLT = 32 * NL;      // loader threads
constexpr int CG_PITCH = ROWS * 16 + 16;   // bytes per landed dz column group (16 rows x 16 B + pad)
constexpr int MAX_L = 6, MAX_SB = 6, MAX_SA = 8;
constexpr int SMEM_MAX = 232448;
// Bottleneck probe (scripts/dts_probe.sh, -DDGNN_DTS_PROBE=mask): 1 skip the
// MMAs, 2 loaders zero-fill instead of reading HBM, 4 promotion without the
// slot update, 8 A converters skip the TMEM stores.  Always 0 in the library.
#ifndef DGNN_DTS_PROBE
#define DGNN_DTS_PROBE 0
#endif
constexpr int PROBE = DGNN_DTS_PROBE;
}  // namespace dts

struct DtsShape {
    int M, mt, N, K4, atoms_b, b_half, bstage, a_land, b_land, land, acc_cols, nacc, a_base, sa, sb, nl;
};

__host__ __device__ inline DtsShape dts_shape(int hp, int kx) {
    DtsShape s;
    s.M = 4 * hp;
    s.mt = s.M / 128;
    s.N = (kx + hp + 31) / 32 * 32;
    s.K4 = (kx + hp) / 4;
    s.atoms_b = s.N / 32;
    s.b_half = 4 * s.atoms_b * 512;
    s.bstage = 2 * s.b_half;
    s.a_land = (s.M / 4) * dts::CG_PITCH;
    s.b_land = dts::ROWS * s.N * 4;
    s.land = s.a_land + s.b_land;
    s.acc_cols = s.mt * s.N;
    // TMEM: accumulator(s), then the A stages (mt tiles x (16 hi + 16 lo) columns each)
    s.nacc = 2 * s.acc_cols + 2 * 32 * s.mt <= 512 ? 2 : 1;
    s.a_base = s.nacc * s.acc_cols;
    s.sa = (512 - s.a_base) / (32 * s.mt);
    if (s.sa > dts::MAX_SA) s.sa = dts::MAX_SA;
    // shared memory: B operand stages (1024-aligned) then the landing ring
    const int avail = dts::SMEM_MAX - 1024 - 1024;
    s.sb = 4;
    s.nl = (avail - s.sb * s.bstage) / s.land;
    if (s.nl > dts::MAX_L) s.nl = dts::MAX_L;
    while (s.nl < 4 && s.sb > 3) {
        --s.sb;
        s.nl = (avail - s.sb * s.bstage) / s.land;
    }
    return s;
}

struct DtsBars {
    uint64_t lfull[dts::MAX_L], lempty[dts::MAX_L], afull[dts::MAX_SA], aempty[dts::MAX_SA], bfull[dts::MAX_SB],
        bempty[dts::MAX_SB], accfull[2], accempty[2];
    uint32_t tmem;
};

// A K-major from TMEM, B MN-major (bit 16), tf32, fp32 D
__host__ __device__ constexpr uint32_t idesc_tf32_ts(int M, int N) { return idesc_tf32(M, N) | (1u << 16); }

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
        :: "r"(tmem_d), "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15, %16};"
                 :: "r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]),
                    "f"(v[7]), "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
                    "f"(v[15]) : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void cp_async16_hint(uint32_t dst, const void* src, uint32_t src_bytes, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;"
                 :: "r"(dst), "l"(src), "r"(src_bytes), "l"(pol) : "memory");
}

__device__ __forceinline__ float lds32(uint32_t saddr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr) : "memory");
    return v;
}

// (as dw_tc.cu) byte offset of (row r in stage, column c) in one MN-major half
__device__ __forceinline__ uint32_t dts_mn_off(int r, int c, int atoms) {
    const int g = r >> 2, r4 = r & 3, j = c >> 5, e = c & 31;
    return (uint32_t)((g * atoms + j) * 512 + r4 * 128 + ((((e >> 3) ^ r4) & 3) << 5) + ((e & 7) << 2));
}

template <int HP>
__global__ void __launch_bounds__(dts::THREADS, 1) lstm_dw_ts_kernel(int64_t rows, int64_t np, int kx,
                                                                   const float* __restrict__ x, int64_t ldx,
                                                                   const float* __restrict__ y,
                                                                   const float* __restrict__ h0,
                                                                   const float* __restrict__ dz,
                                                                   float* __restrict__ slots,
                                                                   double* __restrict__ dbs) {
    constexpr int M = 4 * HP;
    constexpr int NBT = 32 * dts::NB;
    constexpr int B_ITEMS = (dts::ROWS * 64 + NBT - 1) / NBT;        // N <= 256
    constexpr int LA_ITEMS = dts::ROWS * (M / 4) / dts::NLT;         // dz chunks per loader thread
    constexpr int LB_ITEMS = (dts::ROWS * 64 + dts::NLT - 1) / dts::NLT;
    const DtsShape S = dts_shape(HP, kx);
    const int K = kx + HP;

    extern __shared__ uint8_t dts_smem_raw[];
    const uint32_t raw = smem_u32(dts_smem_raw);
    uint8_t* base = dts_smem_raw + ((1024 - (raw & 1023)) & 1023);
    const uint32_t sb = smem_u32(base);
    const uint32_t land0 = sb + S.sb * S.bstage;
    DtsBars* bars = reinterpret_cast<DtsBars*>(base + S.sb * S.bstage + S.nl * S.land);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == dts::MMA_WARP) tmem_alloc(&bars->tmem, 512);
    if (threadIdx.x == 0) {
        for (int i = 0; i < S.nl; ++i) {
            mbar_init(&bars->lfull[i], dts::NLT);
            mbar_init(&bars->lempty[i], 4 * S.mt + dts::NB);
        }
        for (int i = 0; i < S.sa; ++i) {
            mbar_init(&bars->afull[i], 4 * S.mt);
            mbar_init(&bars->aempty[i], 1);
        }
        for (int i = 0; i < S.sb; ++i) {
            mbar_init(&bars->bfull[i], dts::NB);
            mbar_init(&bars->bempty[i], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->accfull[a], 1);
            mbar_init(&bars->accempty[a], dts::NEPI);
        }
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();

    const int64_t per = cdiv(cdiv(rows, gridDim.x), dts::ROWS) * dts::ROWS;
    const int64_t r_begin = blockIdx.x * per;
    const int64_t r_end = min(rows, r_begin + per);
    const int nst = r_end > r_begin ? (int)cdiv(r_end - r_begin, dts::ROWS) : 0;
    const int period_st = dts::PERIOD / dts::ROWS;
    const int nper = (nst + period_st - 1) / period_st;
    float* slot = slots + (size_t)blockIdx.x * M * S.N;   // [N][M]

    if (warp < dts::NA) {
        // A converter: gate column j of tile m, TMEM lane quarter q = warp % 4
        // (hp = 32: one M tile, warps 4..7 idle)
        const int q = warp & 3, m = warp >> 2;
        if (m < S.mt) {
            const int j = 128 * m + 32 * q + lane;
            const uint32_t lane_off = (uint32_t)(32 * q) << 16;
            const uint32_t col_src = (uint32_t)((j >> 2) * dts::CG_PITCH + (j & 3) * 4);
            double db = 0.0;
            for (int g = 0; g < nst; ++g) {
                const int l = g % S.nl, s = g % S.sa;
                const int u = g / S.sa;
                if (u >= 1) mbar_wait(&bars->aempty[s], (u - 1) & 1);
                mbar_wait(&bars->lfull[l], (g / S.nl) & 1);
                const uint32_t src = land0 + l * S.land + col_src;
                float hi[dts::ROWS], lo[dts::ROWS];
#pragma unroll
                for (int i = 0; i < dts::ROWS; ++i) {
                    const float v = lds32(src + 16 * i);
                    hi[i] = tf32_hi(v);
                    lo[i] = v - hi[i];
                    db += v;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->lempty[l]);
                fence_after();
                const uint32_t col = bars->tmem + lane_off + S.a_base + s * 32 * S.mt + 32 * m;
                if (!(dts::PROBE & 8)) {
                    tmem_st16(col, hi);
                    tmem_st16(col + 16, lo);
                    tmem_wait_st();
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->afull[s]);
            }
            dbs[(size_t)blockIdx.x * M + j] = db;
        }
    } else if (warp < dts::LOAD_WARP) {
        // B converter: landed xcat rows -> hi / lo MN-major tiles
        const int pt = threadIdx.x - 32 * dts::NA;
        const int BVEC = dts::ROWS * S.N / 4;
        int boff_land[B_ITEMS];
        uint32_t boff[B_ITEMS];
        bool bz[B_ITEMS];
#pragma unroll
        for (int i = 0; i < B_ITEMS; ++i) {
            const int idx = pt + NBT * i;
            const int r = idx < BVEC ? idx / (S.N / 4) : 0, c = idx < BVEC ? 4 * (idx % (S.N / 4)) : 0;
            boff_land[i] = idx < BVEC ? (r * S.N + c) * 4 : -1;
            boff[i] = idx < BVEC ? dts_mn_off(r, c, S.atoms_b) : 0u;
            bz[i] = c >= K;     // padding columns: zeros
        }
        for (int g = 0; g < nst; ++g) {
            const int l = g % S.nl, s = g % S.sb;
            const int u = g / S.sb;
            if (u >= 1) mbar_wait(&bars->bempty[s], (u - 1) & 1);
            mbar_wait(&bars->lfull[l], (g / S.nl) & 1);
            const uint32_t src = land0 + l * S.land + S.a_land;
            const uint32_t b_hi = sb + s * S.bstage, b_lo = b_hi + S.b_half;
            float4 v[B_ITEMS];
#pragma unroll
            for (int i = 0; i < B_ITEMS; ++i)
                v[i] = (boff_land[i] >= 0 && !bz[i]) ? lds128(src + boff_land[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->lempty[l]);
#pragma unroll
            for (int i = 0; i < B_ITEMS; ++i) {
                if (boff_land[i] >= 0) {
                    float4 hi, lo;
                    split4(v[i], hi, lo);
                    sts128(b_hi + boff[i], hi);
                    sts128(b_lo + boff[i], lo);
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->bfull[s]);
        }
    } else if (warp < dts::MMA_WARP) {
        // loaders: cp.async of stage g's raw rows into landing slot g % nl
        const int pt = threadIdx.x - 32 * dts::LOAD_WARP;
        const uint64_t pol = l2_policy_evict_first();   // operands are read once
        // dz: chunk idx = pt + NLT i -> stage row idx % 16, column group idx / 16
        const int arow = pt % dts::ROWS;
        int64_t ct = r_begin / np, cv = r_begin - ct * np + arow;
        while (cv >= np) {
            cv -= np;
            ++ct;
        }
        int lb_row[LB_ITEMS], lb_col[LB_ITEMS];
#pragma unroll
        for (int i = 0; i < LB_ITEMS; ++i) {
            const int idx = pt + dts::NLT * i;
            lb_row[i] = idx < dts::ROWS * S.K4 ? idx / S.K4 : -1;
            lb_col[i] = idx < dts::ROWS * S.K4 ? 4 * (idx % S.K4) : 0;
        }
        for (int g = 0; g < nst; ++g) {
            const int l = g % S.nl;
            const int u = g / S.nl;
            if (u >= 1) mbar_wait(&bars->lempty[l], (u - 1) & 1);
            const int64_t r0 = r_begin + (int64_t)g * dts::ROWS;
            const uint32_t dst = land0 + l * S.land;
            {
                const bool ok = r0 + arow < r_end && !(dts::PROBE & 2);
                const int64_t v0 = cv & ~(int64_t)127;
                const int64_t tr = min((int64_t)128, np - v0);
                const float* rowp = dz + (ct * np + v0) * M + (cv - v0) * 4;   // tb_off(cv, 0, M, np)
#pragma unroll
                for (int i = 0; i < LA_ITEMS; ++i) {
                    const int cg = (pt + dts::NLT * i) / dts::ROWS;
                    cp_async16_hint(dst + cg * dts::CG_PITCH + arow * 16, ok ? rowp + (int64_t)cg * 4 * tr : dz,
                                    ok ? 16u : 0u, pol);
                }
                cv += dts::ROWS;
                while (cv >= np) {
                    cv -= np;
                    ++ct;
                }
            }
#pragma unroll
            for (int i = 0; i < LB_ITEMS; ++i) {
                if (lb_row[i] >= 0) {
                    const int64_t gr = r0 + lb_row[i];
                    const int c = lb_col[i];
                    const bool ok = gr < r_end && !(dts::PROBE & 2);
                    const float* src = !ok ? x
                                           : (c < kx ? x + gr * ldx + c
                                                     : (gr >= np ? y + (gr - np) * HP + (c - kx) : h0 + gr * HP + (c - kx)));
                    cp_async16_hint(dst + S.a_land + (lb_row[i] * S.N + c) * 4, src, ok ? 16u : 0u, pol);
                }
            }
            cp_async_mbar_arrive(&bars->lfull[l]);
        }
        cp_async_wait<0>();
    } else if (warp == dts::MMA_WARP) {
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32_ts(128, S.N);
            int g = 0;
            for (int p = 0; p < nper; ++p) {
                const int a = S.nacc == 2 ? (p & 1) : 0;
                const int u = S.nacc == 2 ? (p >> 1) : p;
                if (u >= 1) mbar_wait(&bars->accempty[a], (u - 1) & 1);
                fence_after();
                const uint32_t dbase = bars->tmem + a * S.acc_cols;
                const int g_end = min(nst, (p + 1) * period_st);
                for (bool first = true; g < g_end; ++g, first = false) {
                    const int sa = g % S.sa, sbs = g % S.sb;
                    mbar_wait(&bars->afull[sa], (g / S.sa) & 1);
                    mbar_wait(&bars->bfull[sbs], (g / S.sb) & 1);
                    fence_after();
                    const uint32_t abase = bars->tmem + S.a_base + sa * 32 * S.mt;
                    const uint32_t b_hi = sb + sbs * S.bstage, b_lo = b_hi + S.b_half;
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint64_t bh = sdesc_mn(b_hi + 2 * kk * S.atoms_b * 512, 512, S.atoms_b * 512, 1);
                        const uint64_t bl = sdesc_mn(b_lo + 2 * kk * S.atoms_b * 512, 512, S.atoms_b * 512, 1);
                        for (int m = 0; m < S.mt; ++m) {
                            if (dts::PROBE & 1) break;
                            const uint32_t ah = abase + 32 * m + 8 * kk, al = ah + 16;
                            const uint32_t d = dbase + m * S.N;
                            mma_tf32_ts(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                            mma_tf32_ts(d, ah, bl, idesc, 1u);
                            mma_tf32_ts(d, al, bh, idesc, 1u);
                        }
                    }
                    commit(&bars->aempty[sa]);
                    commit(&bars->bempty[sbs]);
                }
                commit(&bars->accfull[a]);
            }
        }
        __syncwarp();
    } else {
        // promotion: TMEM period sum -> fp32 slot[k][j] (round to nearest)
        const int q = warp & 3;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const uint64_t keep = l2_policy_evict_last();   // the CTA slot stays in L2
        for (int p = 0; p < nper; ++p) {
            const int a = S.nacc == 2 ? (p & 1) : 0;
            const int u = S.nacc == 2 ? (p >> 1) : p;
            mbar_wait(&bars->accfull[a], u & 1);
            fence_after();
            for (int m = 0; m < S.mt; ++m) {
                const int j = m * 128 + 32 * q + lane;
                constexpr int GR = 4;
                for (int c0 = 0; c0 < S.N; c0 += 8 * GR) {
                    float v[GR][8];
#pragma unroll
                    for (int ci = 0; ci < GR; ++ci)
                        if (c0 + 8 * ci < S.N) tmem_ld8(bars->tmem + lane_off + a * S.acc_cols + m * S.N + c0 + 8 * ci, v[ci]);
                    tmem_wait_ld();
#pragma unroll
                    for (int ci = 0; ci < GR; ++ci)
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            if (c0 + 8 * ci < S.N && !(dts::PROBE & 4)) red_add(slot + (size_t)(c0 + 8 * ci + t) * M + j, v[ci][t], keep);
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->accempty[a]);
        }
    }
    fence_before();
    __syncthreads();
    if (warp == dts::MMA_WARP) tmem_dealloc(bars->tmem, 512);
}

// fp64 fixed-order reduction of the CTA slots (dw_tc.cu)
__global__ void dw_reduce_kernel(int nct, int M, int N, int K, const float* __restrict__ slots,
                                 const double* __restrict__ dbs, double* __restrict__ gw, int64_t ldg,
                                 double* __restrict__ gb);

template <int HP>
int lstm_dw_ts_t(int64_t rows, int64_t np, int kx, const float* x, int64_t ldx, const float* y, const float* h0,
                 const float* dz, double* gw, double* gb, void* ws, size_t ws_bytes, cudaStream_t st) {
    const DtsShape S = dts_shape(HP, kx);
    if (S.N > 256 || S.sa < 2 || S.sb < 3 || S.nl < 2) {
        set_error("lstm_weight_grad_ts: kx + hp = %d too wide", kx + HP);
        return DGNN_EUNSUPPORTED;
    }
    const int grid = num_sms();
    const size_t need = (size_t)grid * S.M * S.N * sizeof(float) + (size_t)grid * S.M * sizeof(double);
    if (ws_bytes < need) {
        set_error("lstm_weight_grad_ts: workspace too small");
        return DGNN_EWORKSPACE;
    }
    float* slots = reinterpret_cast<float*>(ws);
    double* dbs = reinterpret_cast<double*>(slots + (size_t)grid * S.M * S.N);
    cudaMemsetAsync(slots, 0, (size_t)grid * S.M * S.N * sizeof(float), st);
    auto k = lstm_dw_ts_kernel<HP>;
    const size_t smem = (size_t)S.sb * S.bstage + (size_t)S.nl * S.land + 1024 + sizeof(DtsBars);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch();
    k<<<grid, dts::THREADS, smem, st>>>(rows, np, kx, x, ldx, y, h0, dz, slots, dbs);
    const int K = kx + HP;
    const int64_t tot = (int64_t)S.M * K + S.M;
    note_launch();
    dw_reduce_kernel<<<(unsigned)cdiv(tot * 32, 256), 256, 0, st>>>(grid, S.M, S.N, K, slots, dbs, gw, S.M, gb);
    return launch_status("lstm_weight_grad_ts");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

int dgnn_lstm_weight_grad_ts(int64_t rows, int64_t np, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                             const float* h_out, const float* h0, const float* dz, double* gwcat, double* gb,
                             void* workspace, size_t workspace_bytes, void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && np > 0 && kx % 4 == 0 && ldx % 4 == 0, "lstm_weight_grad_ts: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 32: return lstm_dw_ts_t<32>(rows, np, kx, x, ldx, h_out, h0, dz, gwcat, gb, workspace, workspace_bytes, st);
        case 64: return lstm_dw_ts_t<64>(rows, np, kx, x, ldx, h_out, h0, dz, gwcat, gb, workspace, workspace_bytes, st);
    }
    set_error("lstm_weight_grad_ts: unsupported hp %d", hp);
    return DGNN_EUNSUPPORTED;
}

}  // extern "C"
