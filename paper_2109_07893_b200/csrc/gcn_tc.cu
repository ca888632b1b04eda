// K3 on tcgen05: fused sparse aggregation + dense GCN transform + ReLU
// (core.py:142-161 spmm, training.py:342-367 GCN cells, models.py:200-212).
//
//   s = Ahat x (CSR gather), q = s W, r = relu([s, q]) (skip-concat) | relu(q)
//
// The aggregation is an HBM-bound gather; the transform is a GEMM.  The
// SIMT kernel in spmm.cu does the transform with shared-memory broadcast
// FMAs and is L1-bound at ~22% of HBM.  Here the transform runs on the
// tensor cores, so the SM only gathers:
//
//   warps 0..19  gather: per 128-row tile, one lane group (FP/4 lanes, a
//                float4 each) per row; neighbour rows are fetched with the
//                row's indices read from shared memory, s / relu(s) stored
//                straight from registers (coalesced), and s is split to tf32
//                hi/lo into the SW64 K-major A tile;
//   warp 20      index loader: stages the tile's rowptr slice and its
//                col/val range into shared memory two tiles ahead, so the
//                gather issues the x loads after one latency, not three;
//   warp 21      MMA issuer (one lane): 3xTF32, M = 128, N = HP, K = FP,
//                W (hi/lo, K-major) resident in shared memory;
//   warps 22..25 epilogue: TMEM -> ReLU -> per-warp shared-memory transpose
//                -> row-contiguous stores of relu(q).
//
// Persistent grid (one CTA per SM), 2-stage A ring, 3-stage index ring,
// 2 TMEM accumulators.  FP in {16, 32, 64}, HP in {16, 32, 64}.
//
// BWD instance (K4 rows, training.py:347-350, 359-367): the same pipeline
// computes ds = dpre[:, :F] (skip) + dq W^T with dpre = dr (.) [r > 0] and
// dq = dpre[:, F:] (skip) | dpre (plain): the gather warps load dq rows
// (masked on the fly, no aggregation) as the K-major A tile (K = hidden),
// the W image holds B[f][h] = W[f][h] (N = F), and the epilogue adds the
// skip term dpre[:, :F] in its row-contiguous store pass.
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

__device__ __forceinline__ void fma4(float4& a, float s, const float4& b) {
    a.x = fmaf(s, b.x, a.x);
    a.y = fmaf(s, b.y, a.y);
    a.z = fmaf(s, b.z, a.z);
    a.w = fmaf(s, b.w, a.w);
}

namespace gtc {
// BWD bottleneck probe (scripts/gtb_probe.sh builds with -DDGNN_GTB_PROBE=mask):
// 1 epilogue without the skip-term loads, 2 gathers without the mask loads,
// 4 epilogue without global stores, 8 gathers without any HBM load.
#ifndef DGNN_GTB_PROBE
#define DGNN_GTB_PROBE 0
#endif
constexpr int PROBE = DGNN_GTB_PROBE;
constexpr int BM = 128;
#ifndef DGNN_GTC_NGATHER
#define DGNN_GTC_NGATHER 20
#endif
constexpr int NGATHER = DGNN_GTC_NGATHER, IDX_WARP = NGATHER, MMA_WARP = NGATHER + 1, EPI0 = NGATHER + 2, NEPI = 4;
constexpr int THREADS = 32 * (EPI0 + NEPI);
constexpr int ASTAGES = 3, ISTAGES = 4;   // maxima (GtcLayout::AST / IST per width)
constexpr int ECAP = 1024;   // edges per tile staged in shared memory (else read from global)
}  // namespace gtc

struct GtcBars {
    uint64_t full[gtc::ASTAGES], empty[gtc::ASTAGES], ifull[gtc::ISTAGES], iempty[gtc::ISTAGES], accfull[2],
        accempty[2], skipready[2], skipfree[2];
    uint32_t tmem;
    int32_t claim[gtc::ISTAGES];   // row-chunk claim counters (monotonic)
};

struct GtcIdx {            // one index stage
    int32_t rp[gtc::BM + 4];   // rowptr slice, rebased to ebase
    int32_t ebase, spill;
    int32_t col[gtc::ECAP];
    float val[gtc::ECAP];
};

template <int FP, int HP>
struct GtcLayout {
    static constexpr int KCH = FP / 16;                    // K chunks of 16
    static constexpr int A_HALF = KCH * gtc::BM * 64;      // hi (or lo) of one A stage
    static constexpr int A_STAGE = 2 * A_HALF;
    static constexpr int B_HALF = KCH * HP * 64;
    static constexpr int EPI_BUF = 32 * HP * 4;            // per epilogue warp
    // A stages: 3 for narrow operands (more tiles' gathers in flight), 2 at FP = 64
    static constexpr int AST = FP <= 32 ? 3 : 2;
    static constexpr int IST = AST + 1;
    static constexpr int OFF_B = AST * A_STAGE;
    static constexpr int OFF_EPI = OFF_B + 2 * B_HALF;
    static constexpr int OFF_IDX = OFF_EPI + gtc::NEPI * EPI_BUF;
    static constexpr int OFF_BARS = OFF_IDX + IST * (int)sizeof(GtcIdx);
    static constexpr int BYTES = OFF_BARS + (int)sizeof(GtcBars) + 1024;
    static constexpr int TMEM_COLS = 2 * HP <= 32 ? 32 : (2 * HP <= 64 ? 64 : 128);
};

template <int FP, int HP, bool SKIP, bool AGG, bool BWD>
__global__ void __launch_bounds__(gtc::THREADS, 1) gcn_fwd_tc_kernel(
    int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col, const float* __restrict__ val,
    dgnn_frame x, const float* __restrict__ w, dgnn_frame s_out, dgnn_frame r_out, dgnn_frame mk) {
    static_assert(!(BWD && AGG), "the backward instance has no aggregation");
    using L = GtcLayout<FP, HP>;
    // BWD: x = dr, mk = r (mask source), r_out = ds; dq sits at column
    // offset F (= HP) of dr / r in the skip layer
    constexpr int DQ_OFF = (BWD && SKIP) ? HP : 0;
    constexpr int G = FP / 4;              // lanes per row
    constexpr int RW = 32 / G;             // rows per warp pass
    extern __shared__ uint8_t gtc_smem_raw[];
    const uint32_t raw = smem_u32(gtc_smem_raw);
    uint8_t* base = gtc_smem_raw + ((1024 - (raw & 1023)) & 1023);
    const uint32_t sb = smem_u32(base);
    GtcIdx* idx = reinterpret_cast<GtcIdx*>(base + L::OFF_IDX);
    GtcBars* bars = reinterpret_cast<GtcBars*>(base + L::OFF_BARS);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (int)cdiv(n, gtc::BM);

    // W image: B[j][k] = W[k][j] (forward; BWD: W[j][k]), tf32 hi / lo, SW64
    // K-major chunks of 16 k
    for (int i = threadIdx.x; i < HP * FP / 4; i += gtc::THREADS) {
        const int j = i / (FP / 4), k4 = i % (FP / 4);
        const int k = 4 * k4;
        const float4 v = BWD ? *reinterpret_cast<const float4*>(w + j * FP + k)
                             : make_float4(w[(k + 0) * HP + j], w[(k + 1) * HP + j], w[(k + 2) * HP + j],
                                           w[(k + 3) * HP + j]);
        float4 hi, lo;
        split4(v, hi, lo);
        const uint32_t o = (uint32_t)((k / 16) * HP * 64) + sw64(j, (k % 16) / 4);
        sts128(sb + L::OFF_B + o, hi);
        sts128(sb + L::OFF_B + L::B_HALF + o, lo);
    }
    if (warp == gtc::MMA_WARP) tmem_alloc(&bars->tmem, L::TMEM_COLS);
    if (threadIdx.x == 0) {
        for (int s = 0; s < L::AST; ++s) {
            mbar_init(&bars->full[s], gtc::NGATHER);
            mbar_init(&bars->empty[s], 1);
            bars->claim[s] = 0;
            if (s == 0)
                for (int k = L::AST; k < L::IST; ++k) bars->claim[k] = 0;
        }
        for (int s = 0; s < L::IST; ++s) {
            mbar_init(&bars->ifull[s], 1);
            mbar_init(&bars->iempty[s], gtc::NGATHER);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->accfull[a], 1);
            mbar_init(&bars->accempty[a], gtc::NEPI);
            mbar_init(&bars->skipready[a], 32 * gtc::NGATHER);
            mbar_init(&bars->skipfree[a], gtc::NEPI);
        }
        fence_mbar_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();

    if (warp < gtc::NGATHER) {
        const int sub = lane / G, gl = lane % G;
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it % L::AST, si = it % L::IST;
            const GtcIdx& ix = idx[si];
            if (AGG) mbar_wait_sleep(&bars->ifull[si], (it / L::IST) & 1);
            if (it >= L::AST) mbar_wait_sleep(&bars->empty[s], ((it / L::AST) - 1) & 1);
            const uint32_t a_hi = sb + s * L::A_STAGE, a_lo = a_hi + L::A_HALF;
            const bool spill = AGG && ix.spill;
            // BWD skip: the skip term dpre[:, :F] of this tile's rows goes to ds
            // now; the epilogue adds q on top (RED) once skipready[it & 1]
            // completes.  skipfree keeps the gathers at most one tile ahead of it.
            if (BWD && SKIP && it >= 2) mbar_wait_sleep(&bars->skipfree[it & 1], ((it >> 1) - 1) & 1);
            // two rows per lane group per pass, the first four edges of both
            // in flight together (mean degree is ~2: most rows are one batch)
            const int32_t* cs = spill ? col + ix.ebase : ix.col;
            const float* vs = spill ? val + ix.ebase : ix.val;
            auto xrow = [&](int c) { return __ldg(reinterpret_cast<const float4*>(frame_row<const float>(x, c)) + gl); };
            auto tail = [&](float4& acc, int e, int ee) {   // edges past the first four: the SIMT order
                for (; e + 3 < ee; e += 4) {
                    const int c0 = cs[e], c1 = cs[e + 1], c2 = cs[e + 2], c3 = cs[e + 3];
                    const float v0 = vs[e], v1 = vs[e + 1], v2 = vs[e + 2], v3 = vs[e + 3];
                    const float4 x0 = xrow(c0), x1 = xrow(c1), x2 = xrow(c2), x3 = xrow(c3);
                    fma4(acc, v0, x0);
                    fma4(acc, v1, x1);
                    fma4(acc, v2, x2);
                    fma4(acc, v3, x3);
                }
                for (; e < ee; ++e) fma4(acc, vs[e], xrow(cs[e]));
            };
            // Row chunks (2 RW rows: two rows per lane group) are claimed
            // dynamically, so warps that drew short rows take more of them
            // and the tile completes together.  Every warp makes exactly one
            // failing claim per tile, so use k of stage s starts its claims
            // at k (NCHUNK + NGATHER): the counter never needs a reset (the
            // A ring's empty[s] keeps every warp within one use of stage s).
            constexpr int CROWS = 2 * RW, NCHUNK = gtc::BM / CROWS;
            const int cslot = s;
            const int cbase = (int)(it / L::AST) * (NCHUNK + gtc::NGATHER);
            for (;;) {
                int chunk = 0;
                if (lane == 0) chunk = atomicAdd(&bars->claim[cslot], 1) - cbase;
                chunk = __shfl_sync(0xffffffffu, chunk, 0);
                if (chunk >= NCHUNK) break;
                const int r = chunk * CROWS + sub, rb = r + RW;
                const int64_t row_a = (int64_t)tile * gtc::BM + r, row_b = (int64_t)tile * gtc::BM + rb;
                const bool oka = row_a < n, okb = rb < gtc::BM && row_b < n;
                float4 acc_a = make_float4(0.f, 0.f, 0.f, 0.f), acc_b = acc_a;
                if constexpr (AGG) {
                    const int ea = oka ? ix.rp[r] : 0, eb = okb ? ix.rp[rb] : 0;
                    int eea = oka ? ix.rp[r + 1] : 0, eeb = okb ? ix.rp[rb + 1] : 0;
                    if (eea - ea > kHubRow) eea = ea;   // hub rows: hub_rows_kernel
                    if (eeb - eb > kHubRow) eeb = eb;
                    float4 xa[4], xb[4];
                    float wa[4], wb[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool ja = ea + j < eea, jb = eb + j < eeb;
                        wa[j] = ja ? vs[ea + j] : 0.f;
                        wb[j] = jb ? vs[eb + j] : 0.f;
                        xa[j] = ja ? xrow(cs[ea + j]) : make_float4(0.f, 0.f, 0.f, 0.f);
                        xb[j] = jb ? xrow(cs[eb + j]) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        fma4(acc_a, wa[j], xa[j]);
                        fma4(acc_b, wb[j], xb[j]);
                    }
                    if (eea - ea > 4) tail(acc_a, ea + 4, eea);
                    if (eeb - eb > 4) tail(acc_b, eb + 4, eeb);
                } else if constexpr (BWD) {
                    auto dqrow = [&](int64_t row) {
                        if (gtc::PROBE & 8) return make_float4(1.f, 0.f, 1.f, 0.f);
                        const float4 g = __ldg(reinterpret_cast<const float4*>(frame_row<const float>(x, row) + DQ_OFF) + gl);
                        const float4 m = (gtc::PROBE & 2) ? g : __ldg(reinterpret_cast<const float4*>(frame_row<const float>(mk, row) + DQ_OFF) + gl);
                        return make_float4(m.x > 0.f ? g.x : 0.f, m.y > 0.f ? g.y : 0.f, m.z > 0.f ? g.z : 0.f,
                                           m.w > 0.f ? g.w : 0.f);
                    };
                    if (oka) acc_a = dqrow(row_a);
                    if (okb) acc_b = dqrow(row_b);
                    if constexpr (SKIP) {
                        auto skip_chunk = [&](int64_t row, int c) {
                            const float4 g = __ldg(reinterpret_cast<const float4*>(frame_row<const float>(x, row)) + c);
                            const float4 m = __ldg(reinterpret_cast<const float4*>(frame_row<const float>(mk, row)) + c);
                            reinterpret_cast<float4*>(frame_row<float>(r_out, row))[c] =
                                make_float4(m.x > 0.f ? g.x : 0.f, m.y > 0.f ? g.y : 0.f, m.z > 0.f ? g.z : 0.f,
                                            m.w > 0.f ? g.w : 0.f);
                        };
                        for (int c = gl; c < HP / 4; c += G) {
                            if (oka) skip_chunk(row_a, c);
                            if (okb) skip_chunk(row_b, c);
                        }
                    }
                } else {
                    if (oka) acc_a = xrow((int)row_a);
                    if (okb) acc_b = xrow((int)row_b);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rr = h ? rb : r;
                    if (rr >= gtc::BM) break;
                    const int64_t row = h ? row_b : row_a;
                    const float4 acc = h ? acc_b : acc_a;
                    if (!BWD && (h ? okb : oka)) {
                        if (s_out.ptr) reinterpret_cast<float4*>(frame_row<float>(s_out, row))[gl] = acc;
                        if (SKIP)
                            reinterpret_cast<float4*>(frame_row<float>(r_out, row))[gl] = make_float4(
                                fmaxf(acc.x, 0.f), fmaxf(acc.y, 0.f), fmaxf(acc.z, 0.f), fmaxf(acc.w, 0.f));
                    }
                    float4 hi, lo;
                    split4(acc, hi, lo);
                    const int k = 4 * gl;
                    const uint32_t o = (uint32_t)((k / 16) * gtc::BM * 64) + sw64(rr, (k % 16) / 4);
                    sts128(a_hi + o, hi);
                    sts128(a_lo + o, lo);
                }
            }
            fence_async_smem();
            if (BWD && SKIP) mbar_arrive(&bars->skipready[it & 1]);   // every lane: releases its ds stores
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&bars->full[s]);
                if (AGG) mbar_arrive(&bars->iempty[si]);
            }
        }
    } else if (warp == gtc::IDX_WARP) {
        if (AGG) {
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int si = it % L::IST;
                if (it >= L::IST) mbar_wait_sleep(&bars->iempty[si], ((it / L::IST) - 1) & 1);
                GtcIdx& ix = idx[si];
                const int64_t r0 = (int64_t)tile * gtc::BM;
                const int nr = (int)min((int64_t)gtc::BM, (int64_t)n - r0);
                // all loads of a stage issued before any store (5 rowptr and up
                // to 2 x 8 edge loads in flight per lane): one round trip to
                // memory per 256 edges, so this warp keeps ahead of the gathers
                const int eb = __ldg(rp + r0);
                {
                    int q[5];
#pragma unroll
                    for (int k = 0; k < 5; ++k) {
                        const int i = lane + 32 * k;
                        q[k] = i <= gtc::BM ? __ldg(rp + r0 + min(i, nr)) : 0;
                    }
#pragma unroll
                    for (int k = 0; k < 5; ++k) {
                        const int i = lane + 32 * k;
                        if (i <= gtc::BM) ix.rp[i] = q[k] - eb;
                    }
                }
                __syncwarp();
                const int ne = ix.rp[nr];
                const bool spill = ne > gtc::ECAP;
                if (!spill) {
                    for (int i0 = 0; i0 < ne; i0 += 32 * 8) {
                        int c8[8];
                        float v8[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int i = i0 + 32 * k + lane;
                            c8[k] = i < ne ? __ldg(col + eb + i) : 0;
                            v8[k] = i < ne ? __ldg(val + eb + i) : 0.f;
                        }
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int i = i0 + 32 * k + lane;
                            if (i < ne) {
                                ix.col[i] = c8[k];
                                ix.val[i] = v8[k];
                            }
                        }
                    }
                }
                if (lane == 0) {
                    ix.ebase = eb;
                    ix.spill = spill;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->ifull[si]);   // release: the stores above happen-before
            }
        }
    } else if (warp == gtc::MMA_WARP) {
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(gtc::BM, HP);
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int s = it % L::AST;
                const uint32_t a = it & 1, u = it >> 1;
                if (u >= 1) mbar_wait_sleep(&bars->accempty[a], (u - 1) & 1);
                mbar_wait_sleep(&bars->full[s], (it / L::AST) & 1);
                fence_after();
                const uint32_t d = bars->tmem + a * HP;
                const uint32_t a_hi = sb + s * L::A_STAGE, a_lo = a_hi + L::A_HALF;
                const uint32_t b_hi = sb + L::OFF_B, b_lo = b_hi + L::B_HALF;
#pragma unroll
                for (int kc = 0; kc < L::KCH; ++kc) {
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint32_t ao = kc * gtc::BM * 64 + 32 * kk, bo = kc * HP * 64 + 32 * kk;
                        const uint64_t ah = sdesc(a_hi + ao, 512, kSW64), al = sdesc(a_lo + ao, 512, kSW64);
                        const uint64_t bh = sdesc(b_hi + bo, 512, kSW64), bl = sdesc(b_lo + bo, 512, kSW64);
                        mma_tf32(d, ah, bh, idesc, (kc == 0 && kk == 0) ? 0u : 1u);
                        mma_tf32(d, ah, bl, idesc, 1u);
                        mma_tf32(d, al, bh, idesc, 1u);
                    }
                }
                commit(&bars->empty[s]);
                commit(&bars->accfull[a]);
            }
        }
        __syncwarp();
    } else {
        // epilogue: warp w owns TMEM lane quarter w % 4 (32 tile rows)
        const int q = warp & 3;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const uint32_t buf = sb + L::OFF_EPI + (warp - gtc::EPI0) * L::EPI_BUF;
        constexpr int CPR = HP / 4;   // 16-byte chunks per row
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const uint32_t a = it & 1, u = it >> 1;
            mbar_wait_sleep(&bars->accfull[a], u & 1);
            fence_after();
#pragma unroll
            for (int c0 = 0; c0 < HP; c0 += 8) {
                float v[8];
                tmem_ld8(bars->tmem + lane_off + a * HP + c0, v);
                tmem_wait_ld();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int c = c0 / 4 + h;
                    sts128(buf + lane * HP * 4 + ((c ^ (lane & 7) % CPR) << 4),
                           BWD ? make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3])
                               : make_float4(fmaxf(v[4 * h], 0.f), fmaxf(v[4 * h + 1], 0.f),
                                             fmaxf(v[4 * h + 2], 0.f), fmaxf(v[4 * h + 3], 0.f)));
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->accempty[a]);
            if (BWD && SKIP) mbar_wait_sleep(&bars->skipready[a], u & 1);
            // row-contiguous stores: 32 / CPR rows per warp instruction
            constexpr int RPI = 32 / CPR;
            const int rr = lane / CPR, c = lane % CPR;
#pragma unroll(BWD ? 8 : 4)
            for (int r0 = 0; r0 < 32; r0 += RPI) {
                const int r = r0 + rr;
                const int64_t row = (int64_t)tile * gtc::BM + 32 * q + r;
                const float4 vv = lds128(buf + r * HP * 4 + ((c ^ (r & 7) % CPR) << 4));
                if (row < n) {
                    float* dst = frame_row<float>(r_out, row) + (BWD ? 0 : (SKIP ? FP : 0)) + 4 * c;
                    if (BWD && SKIP) {
                        if (!(gtc::PROBE & 4)) red_add4(dst, vv);   // ds = dpre[:, :F] (gathers) + q
                    } else {
                        *reinterpret_cast<float4*>(dst) = vv;
                    }
                }
            }
            __syncwarp();
            if (BWD && SKIP && lane == 0) mbar_arrive(&bars->skipfree[a]);
        }
    }
    fence_before();
    __syncthreads();
    if (warp == gtc::MMA_WARP) tmem_dealloc(bars->tmem, L::TMEM_COLS);
}

template <int FP, int HP, bool SKIP, bool AGG, bool BWD = false>
int gcn_fwd_tc_t(int32_t n, const int32_t* rp, const int32_t* col, const float* val, dgnn_frame x, const float* w,
                 dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st, dgnn_frame mk = dgnn_frame{}) {
    using L = GtcLayout<FP, HP>;
    auto k = gcn_fwd_tc_kernel<FP, HP, SKIP, AGG, BWD>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
    const int ntiles = (int)cdiv(n, gtc::BM);
    const int grid = ntiles < persistent_ctas() ? ntiles : persistent_ctas();
    note_launch();
    k<<<grid, gtc::THREADS, L::BYTES, st>>>(n, rp, col, val, x, w, s_out, r_out, mk);
    return launch_status(BWD ? "gcn_backward_rows (tcgen05)" : "gcn_forward (tcgen05)");
}

// dispatch used by dgnn_gcn_forward; returns -1 when the shape has no
// tensor-core instance (the caller then uses the SIMT kernel)
int gcn_fwd_tc(int fp, int hp, bool skip, bool agg, int32_t n, const int32_t* rp, const int32_t* col,
               const float* val, dgnn_frame x, const float* w, dgnn_frame s_out, dgnn_frame r_out, cudaStream_t st) {
#define GTC_CASE(F, H)                                                                                         \
    if (fp == F && hp == H) {                                                                                  \
        if (skip) return agg ? gcn_fwd_tc_t<F, H, true, true>(n, rp, col, val, x, w, s_out, r_out, st)         \
                             : gcn_fwd_tc_t<F, H, true, false>(n, rp, col, val, x, w, s_out, r_out, st);       \
        return agg ? gcn_fwd_tc_t<F, H, false, true>(n, rp, col, val, x, w, s_out, r_out, st)                  \
                   : gcn_fwd_tc_t<F, H, false, false>(n, rp, col, val, x, w, s_out, r_out, st);                \
    }
    GTC_CASE(16, 16) GTC_CASE(16, 32) GTC_CASE(16, 64)
    GTC_CASE(32, 16) GTC_CASE(32, 32) GTC_CASE(32, 64)
    GTC_CASE(64, 16) GTC_CASE(64, 32) GTC_CASE(64, 64)
#undef GTC_CASE
    return -1;
}

// K4 rows on tcgen05: fp = F (MMA N), hp = hidden (MMA K); -1 when the
// shape has no instance (the caller then uses the SIMT kernel)
int gcn_bwd_tc(int fp, int hp, bool skip, int32_t n, dgnn_frame dr, dgnn_frame r, const float* w, dgnn_frame ds,
               cudaStream_t st) {
    const dgnn_frame none{};
#define GTB_CASE(F, H)                                                                                         \
    if (fp == F && hp == H)                                                                                    \
        return skip ? gcn_fwd_tc_t<H, F, true, false, true>(n, nullptr, nullptr, nullptr, dr, w, none, ds, st, r) \
                    : gcn_fwd_tc_t<H, F, false, false, true>(n, nullptr, nullptr, nullptr, dr, w, none, ds, st, r);
    GTB_CASE(16, 16) GTB_CASE(16, 32) GTB_CASE(16, 64)
    GTB_CASE(32, 16) GTB_CASE(32, 32) GTB_CASE(32, 64)
    GTB_CASE(64, 16) GTB_CASE(64, 32) GTB_CASE(64, 64)
#undef GTB_CASE
    return -1;
}

}  // namespace dgnn
