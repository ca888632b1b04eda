// LSTM weight gradients on tcgen05 (the x^T dz, h^T dz, sum dz products of
// training.py:422-424, over every vertex row of every step of a block):
//
//   S[j][k] = sum_r dz[r][j] * xcat[r][k],   xcat[r] = [x_t[v] | h_{t-1}[v]],
//   db[j]   = sum_r dz[r][j],                r = t * NP + v.
//
// Both operands are staged MN-major straight from their row-major HBM
// layout (a 128-byte row segment of 32 columns is one swizzle-atom row), so
// nothing is transposed: A = dz^T (M = 4*HP gate columns, one or two M=128
// tiles), B = xcat^T (N = kx + HP rounded to 32), K = rows.  3xTF32 split as
// in lstm_tc.cu.  One persistent CTA per SM owns a contiguous row range.
//
// Warp-specialised (same scheme as lstm_ws.cu):
//   warps 0..15 producers: load their items of a stage DW_PD stages ahead
//               into registers, split (hi, lo) straight into the swizzled
//               tiles once the slot is free, fold dz into fp64 column sums
//               (db), arrive full[s];
//   warp 16     MMA issuer: 2 x mt x 3 MMAs per 16-row stage;
//   warps 17..20 epilogue: promotion of each finished accumulation period.
//
// tcgen05 fp32 accumulation truncates, so a TMEM accumulator only lives for
// DW_PERIOD rows; then it is promoted (fp32, round-to-nearest) into the CTA's
// own slot in global memory (L2 resident, [N][M] so the promotion reductions
// are coalesced) and restarted.  Two accumulators when 2 mt N <= 512 TMEM
// columns, else one (the MMA then waits for the promotion).  The CTA slots
// are reduced in fp64 in fixed order by a second kernel: deterministic.
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

constexpr int DW_ROWS = 16;      // reduction rows per stage = two 8-row K steps
#ifndef DGNN_DW_PERIOD
#define DGNN_DW_PERIOD 512
#endif
constexpr int DW_PERIOD = DGNN_DW_PERIOD;   // rows per TMEM accumulation period
constexpr int DW_MAX_STAGES = 4;
constexpr int DW_NPROD = 16, DW_MMA_WARP = DW_NPROD, DW_NEPI = 4;
#ifndef DGNN_DW_PD
#define DGNN_DW_PD 2
#endif
constexpr int DW_PD = DGNN_DW_PD;   // stages of operand loads each producer keeps in flight (registers)
// rows ahead of the current stage that the bulk L2 prefetch covers (128-row
// prefetches every 8 stages; 0 = no prefetch)
#ifndef DGNN_DW_PF
#define DGNN_DW_PF 128
#endif
constexpr int DW_THREADS = 32 * (DW_NPROD + 1 + DW_NEPI);
constexpr int DW_SMEM_MAX = 232448;
// Bottleneck probe (scripts/dw_probe.cu, -DDGNN_DW_PROBE=mask): 1 skip MMAs,
// 2 zero-fill operands (no HBM reads), 4 promotion without the slot update,
// 8 producers without the tf32 split.  Always 0 in the library.
#ifndef DGNN_DW_PROBE
#define DGNN_DW_PROBE 0
#endif
constexpr int DW_PROBE = DGNN_DW_PROBE;
// L2 eviction hints on the operand loads (evict-first) and slot reductions
// (evict-last): measured 3% slower at configs[1] shapes (scripts/dw_hint_ab.sh),
// so off; -DDGNN_DW_HINTS=1 for the A/B probe
#ifndef DGNN_DW_HINTS
#define DGNN_DW_HINTS 0
#endif
#if DGNN_DW_PROBE & 16
// probe 16: per-CTA cycles each role spends blocked on its barriers
__device__ unsigned long long dw_prof[kMaxSMs * 8];
#endif
__device__ __forceinline__ void dw_wait(uint64_t* bar, uint32_t parity, long long& acc) {
    if (DW_PROBE & 16) {
        const long long t = clock64();
        mbar_wait(bar, parity);
        acc += clock64() - t;
    } else {
        mbar_wait(bar, parity);
    }
}

struct DwShape {
    int M, mtile, mt, N, atoms_a, atoms_b, a_half, b_half, stage, acc_cols, nacc, tmem_cols, stages;
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
    s.acc_cols = s.mt * s.N;
    s.nacc = 2 * s.acc_cols <= 512 ? 2 : 1;
    const int cols = s.nacc * s.acc_cols;
    s.tmem_cols = cols <= 32 ? 32 : (cols <= 64 ? 64 : (cols <= 128 ? 128 : (cols <= 256 ? 256 : 512)));
    s.stages = (DW_SMEM_MAX - 1024 - 256) / s.stage;
    if (s.stages > DW_MAX_STAGES) s.stages = DW_MAX_STAGES;
    return s;
}

inline size_t dw_smem_bytes(const DwShape& s) { return (size_t)s.stages * s.stage + 1024 + 256; }

struct DwBars {
    uint64_t full[DW_MAX_STAGES], empty[DW_MAX_STAGES], accfull[2], accempty[2];
    uint32_t tmem;
};

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
__global__ void __launch_bounds__(DW_THREADS, 1) lstm_dw_tc_kernel(int64_t rows, int64_t np, int kx,
                                                                   const float* __restrict__ x, int64_t ldx,
                                                                   const float* __restrict__ y,
                                                                   const float* __restrict__ h0,
                                                                   const float* __restrict__ dz,
                                                                   float* __restrict__ slots,
                                                                   double* __restrict__ dbs) {
    constexpr int M = 4 * HP;
    constexpr int NPT = 32 * DW_NPROD;                          // producer threads
    constexpr int A_ITEMS = DW_ROWS * (M / 4) / NPT;            // A float4 items per producer per stage
    constexpr int B_ITEMS = (DW_ROWS * 64 + NPT - 1) / NPT;     // B items (N <= 256)
    const DwShape S = dw_shape(HP, kx);
    const int K = kx + HP;
    const int BVEC = DW_ROWS * S.N / 4;

    extern __shared__ uint8_t dw_smem_raw[];
    const uint32_t raw = smem_u32(dw_smem_raw);
    uint8_t* base = dw_smem_raw + ((1024 - (raw & 1023)) & 1023);
    const uint32_t sb = smem_u32(base);
    DwBars* bars = reinterpret_cast<DwBars*>(base + S.stages * S.stage);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == DW_MMA_WARP) tmem_alloc(&bars->tmem, S.tmem_cols);
    if (threadIdx.x == 0) {
        for (int i = 0; i < S.stages; ++i) {
            mbar_init(&bars->full[i], DW_NPROD);
            mbar_init(&bars->empty[i], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->accfull[a], 1);
            mbar_init(&bars->accempty[a], DW_NEPI);
        }
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();

    // contiguous row range of this CTA (multiple of 16)
    const int64_t per = cdiv(cdiv(rows, gridDim.x), DW_ROWS) * DW_ROWS;
    const int64_t r_begin = blockIdx.x * per;
    const int64_t r_end = min(rows, r_begin + per);
    const int nst = r_end > r_begin ? (int)cdiv(r_end - r_begin, DW_ROWS) : 0;
    const int period_st = DW_PERIOD / DW_ROWS;
    const int nper = (nst + period_st - 1) / period_st;
    float* slot = slots + (size_t)blockIdx.x * M * S.N;   // [N][M]
    double dbacc[4 * (DW_ROWS * (4 * HP / 4) / (32 * DW_NPROD))] = {};
    long long wacc0 = 0, wacc1 = 0;
    const long long t_start = clock64();

    if (warp < DW_NPROD) {
        // Producers: global -> registers (DW_PD stages in flight) -> tf32
        // split -> the SW128_32B hi / lo tiles, and the fp64 column sums of
        // dz (db).  Shared memory sees only the split stores: the operand
        // reads of the 3xTF32 MMAs already take most of its bandwidth, and a
        // raw landing copy plus its re-read measured as the kernel's
        // bottleneck (scripts/dw_probe2.sh: -27% without the split pass).
        const int pt = threadIdx.x;
        const uint64_t pol = l2_policy_evict_first();   // operands are read once
        int acol[A_ITEMS], brow[B_ITEMS], bcol[B_ITEMS];
        uint32_t aoff[A_ITEMS], boff[B_ITEMS];
        // A items: each group of 8 consecutive threads (one shared-memory
        // store wavefront of 16-byte stores) covers 4 rows (one swizzle row
        // group) x 2 column groups (one 32-byte chunk): the 8 stores land in
        // 8 distinct 16-byte bank slots (no conflicts).  A warp covers all 16
        // stage rows of 2 column groups: 2 x 256 contiguous bytes of the
        // tile-blocked dz.  Every A item of a thread is the same stage row.
        const int arow = 4 * ((pt >> 3) & 3) + (pt & 3);
#pragma unroll
        for (int i = 0; i < A_ITEMS; ++i) {
            acol[i] = 8 * ((pt >> 5) + (NPT / 32) * i) + 4 * ((pt >> 2) & 1);
            aoff[i] = mn_off(arow, acol[i], S.atoms_a);
        }
#pragma unroll
        for (int i = 0; i < B_ITEMS; ++i) {
            const int idx = pt + NPT * i;
            brow[i] = idx < BVEC ? idx / (S.N / 4) : -1;
            bcol[i] = idx < BVEC ? 4 * (idx % (S.N / 4)) : 0;
            boff[i] = idx < BVEC ? mn_off(brow[i], bcol[i], S.atoms_b) : 0u;
        }
        // dz is tile-blocked per step (common.cuh tb_off, rows r = t np + v):
        // the (t, v) of this thread's stage row is tracked incrementally
        int64_t ct = r_begin / np, cv = r_begin - ct * np + arow;
        while (cv >= np) {
            cv -= np;
            ++ct;
        }
        // the CTA walks a contiguous row range: every 8 stages, pull the rows
        // 128..255 ahead into L2 with bulk prefetches (x, y / h0 and the
        // tile-blocked dz blocks holding them), so the register loads of a
        // stage (DW_PD stages ahead) hit L2
        const int64_t dz_end = rows * M;
        auto prefetch_rows = [&](int64_t ra) {
            const int64_t rb = min(r_end, ra + 128);
            if (ra >= rb || (DW_PROBE & 2)) return;
            bulk_prefetch_l2(x + ra * ldx, (uint32_t)((rb - ra) * ldx * 4));
            const int64_t ya = ra < np ? ra : ra, yb = rb;
            if (ya < np) bulk_prefetch_l2(h0 + ya * HP, (uint32_t)((min(yb, np) - ya) * HP * 4));
            if (yb > np) bulk_prefetch_l2(y + (max(ya, np) - np) * HP, (uint32_t)((yb - max(ya, np)) * HP * 4));
            const int64_t ta = ra / np, tb = (rb - 1) / np;
            const int64_t da = (ta * np + ((ra - ta * np) & ~(int64_t)127)) * M;
            const int64_t db_ = min(dz_end, (tb * np + (((rb - 1) - tb * np) & ~(int64_t)127) + 128) * M);
            bulk_prefetch_l2(dz + da, (uint32_t)((db_ - da) * 4));
        };
        if (pt == 0 && DGNN_DW_PF)
            for (int a = 0; a < DGNN_DW_PF; a += 128) prefetch_rows(r_begin + a);
        auto load = [&](int g, float4 (&va)[A_ITEMS], float4 (&vb)[B_ITEMS]) {
            const int64_t r0 = r_begin + (int64_t)g * DW_ROWS;
            if (DGNN_DW_PF && pt == 0 && (g & 7) == 0) prefetch_rows(r0 + DGNN_DW_PF);
            const int64_t v0 = cv & ~(int64_t)127;
            const int64_t tr = min((int64_t)128, np - v0);
            const float* rowp = dz + (ct * np + v0) * M + (cv - v0) * 4;   // tb_off(cv, 0, M, np)
            const bool aok = r0 + arow < r_end && !(DW_PROBE & 2);
#pragma unroll
            for (int i = 0; i < A_ITEMS; ++i)
                va[i] = aok ? (DGNN_DW_HINTS ? ldg_stream4(rowp + (int64_t)acol[i] * tr, pol) : ldg_stream4(rowp + (int64_t)acol[i] * tr)) : make_float4(0.f, 0.f, 0.f, 0.f);
            cv += DW_ROWS;
            while (cv >= np) {
                cv -= np;
                ++ct;
            }
#pragma unroll
            for (int i = 0; i < B_ITEMS; ++i) {
                vb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (brow[i] >= 0) {
                    const int64_t gr = r0 + brow[i];
                    const int c = bcol[i];
                    if (gr < r_end && c < K && !(DW_PROBE & 2)) {
                        const float* src = c < kx ? x + gr * ldx + c
                                                  : (gr >= np ? y + (gr - np) * HP + (c - kx) : h0 + gr * HP + (c - kx));
                        vb[i] = DGNN_DW_HINTS ? ldg_stream4(src, pol) : ldg_stream4(src);
                    }
                }
            }
        };
        float4 ra[DW_PD][A_ITEMS], rb[DW_PD][B_ITEMS];
#pragma unroll
        for (int d = 0; d < DW_PD; ++d)
            if (d < nst) load(d, ra[d], rb[d]);
        for (int g0 = 0; g0 < nst; g0 += DW_PD) {
#pragma unroll
            for (int d = 0; d < DW_PD; ++d) {
                const int g = g0 + d;
                if (g >= nst) break;
                const int s = g % S.stages;
                const int j = g / S.stages;
                if (j >= 1) dw_wait(&bars->empty[s], (j - 1) & 1, wacc0);
                const uint32_t a_hi = sb + s * S.stage, a_lo = a_hi + S.a_half;
                const uint32_t b_hi = a_lo + S.a_half, b_lo = b_hi + S.b_half;
#pragma unroll
                for (int i = 0; i < A_ITEMS; ++i) {
                    float4 hi, lo;
                    if (DW_PROBE & 8) {
                        hi = ra[d][i];
                        lo = hi;
                    } else {
                        split4(ra[d][i], hi, lo);
                    }
                    sts128(a_hi + aoff[i], hi);
                    sts128(a_lo + aoff[i], lo);
                    dbacc[4 * i + 0] += ra[d][i].x;
                    dbacc[4 * i + 1] += ra[d][i].y;
                    dbacc[4 * i + 2] += ra[d][i].z;
                    dbacc[4 * i + 3] += ra[d][i].w;
                }
#pragma unroll
                for (int i = 0; i < B_ITEMS; ++i) {
                    if (brow[i] >= 0) {
                        float4 hi, lo;
                        if (DW_PROBE & 8) {
                            hi = rb[d][i];
                            lo = hi;
                        } else {
                            split4(rb[d][i], hi, lo);
                        }
                        sts128(b_hi + boff[i], hi);
                        sts128(b_lo + boff[i], lo);
                    }
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->full[s]);
                if (g + DW_PD < nst) load(g + DW_PD, ra[d], rb[d]);
            }
        }
    } else if (warp == DW_MMA_WARP) {
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32_mn(S.mtile, S.N);
            int g = 0;
            for (int p = 0; p < nper; ++p) {
                const int a = S.nacc == 2 ? (p & 1) : 0;
                const int u = S.nacc == 2 ? (p >> 1) : p;   // use count of accumulator a
                if (u >= 1) dw_wait(&bars->accempty[a], (u - 1) & 1, wacc1);
                fence_after();
                const uint32_t dbase = bars->tmem + a * S.acc_cols;
                const int g_end = min(nst, (p + 1) * period_st);
                for (bool first = true; g < g_end; ++g, first = false) {
                    const int s = g % S.stages;
                    dw_wait(&bars->full[s], (g / S.stages) & 1, wacc0);
                    fence_after();
                    const uint32_t a_hi = sb + s * S.stage, a_lo = a_hi + S.a_half;
                    const uint32_t b_hi = a_lo + S.a_half, b_lo = b_hi + S.b_half;
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint64_t bh = sdesc_mn(b_hi + 2 * kk * S.atoms_b * 512, 512, S.atoms_b * 512, kSW128B32);
                        const uint64_t bl = sdesc_mn(b_lo + 2 * kk * S.atoms_b * 512, 512, S.atoms_b * 512, kSW128B32);
                        for (int m = 0; m < S.mt; ++m) {
                            if (DW_PROBE & 1) break;
                            const uint32_t aoff = (2 * kk * S.atoms_a + m * (S.mtile / 32)) * 512;
                            const uint64_t ah = sdesc_mn(a_hi + aoff, 512, S.atoms_a * 512, kSW128B32);
                            const uint64_t al = sdesc_mn(a_lo + aoff, 512, S.atoms_a * 512, kSW128B32);
                            const uint32_t d = dbase + m * S.N;
                            mma_tf32(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                            mma_tf32(d, ah, bl, idesc, 1u);
                            mma_tf32(d, al, bh, idesc, 1u);
                        }
                    }
                    commit(&bars->empty[s]);
                }
                commit(&bars->accfull[a]);
            }
        }
        __syncwarp();
    } else {
        // promotion: TMEM period sum -> fp32 slot[k][j] (round to nearest);
        // DW_NEPI / 4 warps share a TMEM lane quarter and split the columns
        constexpr int WPQ = DW_NEPI / 4, CS = 8 * WPQ;   // column stride of one warp
        const int e = warp - DW_MMA_WARP - 1;
        const int q = warp & 3, half = e >> 2;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const uint64_t keep = l2_policy_evict_last();   // the CTA slot stays in L2
        for (int p = 0; p < nper; ++p) {
            const int a = S.nacc == 2 ? (p & 1) : 0;
            const int u = S.nacc == 2 ? (p >> 1) : p;
            dw_wait(&bars->accfull[a], u & 1, wacc0);
            fence_after();
            for (int m = 0; m < S.mt; ++m) {
                const int j = m * S.mtile + 32 * q + lane;
                const bool jok = 32 * q + lane < S.mtile;
                // four 8-column chunks per TMEM wait; the slot update is a
                // fire-and-forget reduction (RED.ADD, coalesced over j), so
                // the accumulator is released after the TMEM reads alone.
                // Each slot element is only ever updated by this thread, in
                // period order: the fp32 sum sequence is fixed.
                constexpr int GR = 4;
                for (int c0 = half * 8; c0 < S.N; c0 += CS * GR) {
                    float v[GR][8];
#pragma unroll
                    for (int ci = 0; ci < GR; ++ci)
                        if (c0 + CS * ci < S.N) tmem_ld8(bars->tmem + lane_off + a * S.acc_cols + m * S.N + c0 + CS * ci, v[ci]);
                    tmem_wait_ld();
                    if (jok && !(DW_PROBE & 4)) {
#pragma unroll
                        for (int ci = 0; ci < GR; ++ci)
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                if (c0 + CS * ci < S.N) {
                                    if (DGNN_DW_HINTS) red_add(slot + (size_t)(c0 + CS * ci + t) * M + j, v[ci][t], keep);
                                    else atomicAdd(slot + (size_t)(c0 + CS * ci + t) * M + j, v[ci][t]);
                                }
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->accempty[a]);
        }
    }
#if DGNN_DW_PROBE & 16
    if (lane == 0 && (warp == 0 || warp == 8 || warp == DW_MMA_WARP || warp == DW_MMA_WARP + 1)) {
        const int k = warp == 0 ? 0 : (warp == 8 ? 1 : (warp == DW_MMA_WARP ? 2 : 4));
        dw_prof[blockIdx.x * 8 + k] = wacc0;
        if (warp == DW_MMA_WARP) dw_prof[blockIdx.x * 8 + 3] = wacc1;
        if (warp == 0) dw_prof[blockIdx.x * 8 + 5] = clock64() - t_start;
    }
#endif
    fence_before();
    __syncthreads();
    // db partial: producer threads sharing a column group combine in fixed
    // order (the stage ring is free now)
    // dbred[item][thread][4]: producer thread pt, item i holds column group
    // (pt + NPT i) / 16 of the 16 stage rows pt % 16
    double* dbred = reinterpret_cast<double*>(base);
    if (warp < DW_NPROD) {
#pragma unroll
        for (int i = 0; i < A_ITEMS; ++i)
#pragma unroll
            for (int t = 0; t < 4; ++t) dbred[((size_t)i * NPT + threadIdx.x) * 4 + t] = dbacc[4 * i + t];
    }
    __syncthreads();
    if (threadIdx.x < M / 4) {
        // column group cg = threadIdx.x: its 16 producer slots (one per stage
        // row, the A item mapping above), summed in fixed (row) order
        const int cg = threadIdx.x, cc = cg >> 1, ch = cg & 1;
        const int i = cc / (NPT / 32);
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int r = 0; r < DW_ROWS; ++r) {
            const int pt = 32 * (cc % (NPT / 32)) + 8 * (r >> 2) + 4 * ch + (r & 3);
            for (int jj = 0; jj < 4; ++jj) s4[jj] += dbred[((size_t)i * NPT + pt) * 4 + jj];
        }
        for (int jj = 0; jj < 4; ++jj) dbs[(size_t)blockIdx.x * M + 4 * threadIdx.x + jj] = s4[jj];
    }
    fence_before();
    __syncthreads();
    if (warp == DW_MMA_WARP) tmem_dealloc(bars->tmem, S.tmem_cols);
}

// gw[k][j] += sum_cta slot[cta][k][j] ; gb[j] += sum_cta dbs[cta][j]   (fp64, fixed
// order: one warp per output, lane l sums CTAs l, l + 32, ... then a fixed butterfly)
__global__ void dw_reduce_kernel(int nct, int M, int N, int K, const float* __restrict__ slots,
                                 const double* __restrict__ dbs, double* __restrict__ gw, int64_t ldg,
                                 double* __restrict__ gb) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i < (int64_t)M * K) {
        const int k = (int)(i / M), j = (int)(i % M);
        double s = 0.0;
        for (int c = lane; c < nct; c += 32) s += (double)__ldg(slots + ((size_t)c * N + k) * M + j);
        s = warp_sum(s);
        if (lane == 0) gw[(int64_t)k * ldg + j] += s;
    } else if (i < (int64_t)M * K + M && gb) {
        const int j = (int)(i - (int64_t)M * K);
        double s = 0.0;
        for (int c = lane; c < nct; c += 32) s += dbs[(size_t)c * M + j];
        s = warp_sum(s);
        if (lane == 0) gb[j] += s;
    }
}

template <int HP>
int lstm_dw_tc_t(int64_t rows, int64_t np, int kx, const float* x, int64_t ldx, const float* y, const float* h0,
                 const float* dz, double* gw, double* gb, void* ws, size_t ws_bytes, cudaStream_t st) {
    const DwShape S = dw_shape(HP, kx);
    if (S.acc_cols > 512 || S.N > 256 || S.stages < 3) {
        set_error("lstm_weight_grad_tc: kx + hp = %d too wide", kx + HP);
        return DGNN_EUNSUPPORTED;
    }
    // always one CTA per SM: the CTA row ranges (and so the fp32 period
    // sums) must not depend on dgnn_set_sm_reserve, or results would differ
    // between single- and multi-GPU runs
    const int grid = num_sms();
    const size_t need = (size_t)grid * S.M * S.N * sizeof(float) + (size_t)grid * S.M * sizeof(double);
    if (ws_bytes < need) {
        set_error("lstm_weight_grad_tc: workspace too small");
        return DGNN_EWORKSPACE;
    }
    float* slots = reinterpret_cast<float*>(ws);
    double* dbs = reinterpret_cast<double*>(slots + (size_t)grid * S.M * S.N);
    // slots accumulate period sums by reduction: start from zero
    cudaMemsetAsync(slots, 0, (size_t)grid * S.M * S.N * sizeof(float), st);
    auto k = lstm_dw_tc_kernel<HP>;
    const size_t smem = dw_smem_bytes(S);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch();
    k<<<grid, DW_THREADS, smem, st>>>(rows, np, kx, x, ldx, y, h0, dz, slots, dbs);
    const int K = kx + HP;
    const int64_t tot = (int64_t)S.M * K + S.M;
    note_launch();
    dw_reduce_kernel<<<(unsigned)cdiv(tot * 32, 256), 256, 0, st>>>(grid, S.M, S.N, K, slots, dbs, gw, S.M, gb);
    return launch_status("lstm_weight_grad_tc");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

size_t dgnn_lstm_weight_grad_tc_workspace(int32_t kx, int32_t hp) {
    const DwShape S = dw_shape(hp, kx);
    return (size_t)num_sms() * S.M * S.N * sizeof(float) + (size_t)num_sms() * S.M * sizeof(double) + 256;
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
