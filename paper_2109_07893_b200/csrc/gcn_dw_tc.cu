// GCN weight gradient on tcgen05 (training.py:365 skip cell, training.py:350
// plain cell): the sum over every vertex row of one snapshot of
//
//   dW[f][h] += sum_r s[r][f] * dq[r][h],   dq = dr[:, off:] (.) [r[:, off:] > 0],
//
// off = F for the skip-concat layer (cd-gcn), 0 for the plain layer.  The
// SIMT split-K GEMM in dense.cu (tn_partial) is latency bound at ~1.5 TB/s;
// here the reduction runs on the tensor pipe and the SM only moves bytes.
//
// D = dq^T s: A = dq^T (M = 64 or 128 hidden columns, zero-padded), B = s^T
// (N = F rounded up to 32), K = rows.  Both operands are staged MN-major
// straight from their row-major HBM frames (SWIZZLE_128B_BASE32B atoms, as
// in dw_tc.cu), 3xTF32.
//
//   warps 0..15 loaders (16: 14% faster than 8 at configs[1], scripts/gdw_probe.sh):
//               cp.async the raw fp32 rows of a 32-row stage (dr and
//               r of the dq columns into the A hi / mask areas, s into B hi),
//               completion on landed[s].  Every thread keeps one 4-column
//               group and steps over rows, so its shared-memory offsets are
//               fixed and a row address costs one multiply-add;
//   warps 16..19 converters: dq = dr (.) [r > 0], tf32 split in place (hi, lo);
//   warp 20     MMA issuer: 4 K steps x 3 MMAs per stage into the TMEM
//               accumulator of the current 512-row period;
//   warps 21..24 promotion: each finished period is added (fp32, RED) into the
//               CTA's own slot; a second kernel reduces the slots in fp64 in
//               fixed order -- deterministic, independent of the SM reserve.
//
// M = 64 accumulators live in TMEM lanes (m % 16) + 32 (m / 16) (the
// half-subpartition layout of cta_group::1 M = 64).
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

namespace gdw {
constexpr int ROWS = 32;          // reduction rows per stage (4 MMA K steps of 8)
constexpr int PERIOD = 512;       // rows per TMEM accumulation period
constexpr int MAX_STAGES = 6;
#ifndef DGNN_GDW_NLOAD
#define DGNN_GDW_NLOAD 16
#endif
#ifndef DGNN_GDW_NCONV
#define DGNN_GDW_NCONV 4
#endif
constexpr int NLOAD = DGNN_GDW_NLOAD, NCONV = DGNN_GDW_NCONV, MMA_WARP = NLOAD + NCONV, NEPI = 4;
constexpr int THREADS = 32 * (NLOAD + NCONV + 1 + NEPI);
constexpr int SMEM_MAX = 232448;
}  // namespace gdw

struct GdwShape {
    int MA, N, atoms_a, atoms_b, a_half, b_half, stage, stages, tmem_cols;
};

__host__ __device__ inline GdwShape gdw_shape(int ma, int fp, int rows = gdw::ROWS) {
    GdwShape s;
    s.MA = ma;
    s.N = (fp + 31) / 32 * 32;
    s.atoms_a = s.MA / 32;
    s.atoms_b = s.N / 32;
    s.a_half = (rows / 4) * s.atoms_a * 512;
    s.b_half = (rows / 4) * s.atoms_b * 512;
    s.stage = 3 * s.a_half + 2 * s.b_half;   // A hi | A lo | mask | B hi | B lo
    s.stages = (gdw::SMEM_MAX - 1024 - 256) / s.stage;
    if (s.stages > gdw::MAX_STAGES) s.stages = gdw::MAX_STAGES;
    const int cols = 2 * s.N;
    s.tmem_cols = cols <= 32 ? 32 : (cols <= 64 ? 64 : (cols <= 128 ? 128 : 256));
    return s;
}

struct GdwBars {
    uint64_t landed[gdw::MAX_STAGES], full[gdw::MAX_STAGES], empty[gdw::MAX_STAGES], accfull[2], accempty[2];
    uint32_t tmem;
};

// byte offset of (row r of the stage, column c) in an MN-major operand half:
// [K group of 4 rows][32-column atom][512 B], 32-byte granules swizzled by r % 4
__device__ __forceinline__ uint32_t gdw_off(int r, int c, int atoms) {
    const int g = r >> 2, r4 = r & 3, j = c >> 5, e = c & 31;
    return (uint32_t)((g * atoms + j) * 512 + r4 * 128 + ((((e >> 3) ^ r4) & 3) << 5) + ((e & 7) << 2));
}

__device__ __forceinline__ const float* gdw_row(const dgnn_frame& f, int32_t i) {
    if (f.rows_per_slab <= 0 || i < f.rows_per_slab) return reinterpret_cast<const float*>(f.ptr) + (int64_t)i * f.ld;
    const int32_t rps = (int32_t)f.rows_per_slab;
    const int32_t s = i / rps, r = i - s * rps;
    return reinterpret_cast<const float*>(f.ptr) + (int64_t)s * f.slab_stride + (int64_t)r * f.ld;
}

// R: reduction rows per stage -- 64 for narrow operands (fp <= 32, M = 64),
// so a stage still moves >= 12 KB per cp.async batch
template <int MA, int R>
__global__ void __launch_bounds__(gdw::THREADS, 1) gcn_dw_tc_kernel(int32_t rows, int fp, int hp, int off,
                                                                    dgnn_frame s_in, dgnn_frame dr, dgnn_frame rk,
                                                                    float* __restrict__ slots) {
    const GdwShape S = gdw_shape(MA, fp, R);
    extern __shared__ uint8_t gdw_smem_raw[];
    const uint32_t raw = smem_u32(gdw_smem_raw);
    uint8_t* base = gdw_smem_raw + ((1024 - (raw & 1023)) & 1023);
    const uint32_t sb = smem_u32(base);
    GdwBars* bars = reinterpret_cast<GdwBars*>(base + S.stages * S.stage);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // zero every stage once: padded columns (h >= hp, f >= fp) are never
    // written again and must read as 0 in every MMA
    for (int i = threadIdx.x; i < S.stages * S.stage / 16; i += gdw::THREADS)
        sts128(sb + 16 * i, make_float4(0.f, 0.f, 0.f, 0.f));
    if (warp == gdw::MMA_WARP) tmem_alloc(&bars->tmem, S.tmem_cols);
    if (threadIdx.x == 0) {
        for (int i = 0; i < S.stages; ++i) {
            mbar_init(&bars->landed[i], 32 * gdw::NLOAD);
            mbar_init(&bars->full[i], gdw::NCONV);
            mbar_init(&bars->empty[i], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->accfull[a], 1);
            mbar_init(&bars->accempty[a], gdw::NEPI);
        }
        fence_mbar_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();

    // contiguous row range of this CTA (multiple of the stage rows)
    const int64_t per = cdiv(cdiv(rows, gridDim.x), R) * R;
    const int64_t r_begin = blockIdx.x * per;
    const int64_t r_end = min((int64_t)rows, r_begin + per);
    const int nst = r_end > r_begin ? (int)cdiv(r_end - r_begin, R) : 0;
    constexpr int PST = gdw::PERIOD / R;
    const int nper = (nst + PST - 1) / PST;
    const int ga = hp / 4, gb = fp / 4;   // real 4-column groups of A (dq) and B (s)

    if (warp < gdw::NLOAD) {
        // thread -> (fixed column group, first row, row step); ga / gb are
        // powers of two dividing the loader thread count (host-checked)
        constexpr int NLT = 32 * gdw::NLOAD;
        const int lt = threadIdx.x;
        const int ca = 4 * (lt % ga), ra = lt / ga, rsa = NLT / ga;
        const int cb = 4 * (lt % gb), rb = lt / gb, rsb = NLT / gb;
        const uint32_t aoff0 = gdw_off(ra & (R - 1), ca, S.atoms_a), astep = (uint32_t)(rsa / 4) * S.atoms_a * 512;
        const uint32_t boff0 = gdw_off(rb & (R - 1), cb, S.atoms_b), bstep = (uint32_t)(rsb / 4) * S.atoms_b * 512;
        for (int g = 0; g < nst; ++g) {
            const int s = g % S.stages;
            const int j = g / S.stages;
            if (j >= 1) mbar_wait(&bars->empty[s], (j - 1) & 1);
            const int64_t r0 = r_begin + (int64_t)g * R;
            const uint32_t a_hi = sb + s * S.stage, mk = a_hi + 2 * S.a_half, b_hi = mk + S.a_half;
            uint32_t o = aoff0;
            for (int r = ra; r < R; r += rsa, o += astep) {
                const int64_t gr = r0 + r;
                const bool ok = gr < r_end;
                const float* pd = ok ? gdw_row(dr, (int32_t)gr) + off + ca : reinterpret_cast<const float*>(dr.ptr);
                const float* pm = ok ? gdw_row(rk, (int32_t)gr) + off + ca : reinterpret_cast<const float*>(rk.ptr);
                cp_async16(a_hi + o, pd, ok ? 16u : 0u);
                cp_async16(mk + o, pm, ok ? 16u : 0u);
            }
            o = boff0;
            for (int r = rb; r < R; r += rsb, o += bstep) {
                const int64_t gr = r0 + r;
                const bool ok = gr < r_end;
                const float* ps = ok ? gdw_row(s_in, (int32_t)gr) + cb : reinterpret_cast<const float*>(s_in.ptr);
                cp_async16(b_hi + o, ps, ok ? 16u : 0u);
            }
            cp_async_mbar_arrive(&bars->landed[s]);
        }
        cp_async_wait<0>();
    } else if (warp < gdw::MMA_WARP) {
        constexpr int NCT = 32 * gdw::NCONV;
        const int ct = threadIdx.x - 32 * gdw::NLOAD;
        const int ca = 4 * (ct % ga), ra = ct / ga, rsa = NCT / ga;
        const int cb = 4 * (ct % gb), rb = ct / gb, rsb = NCT / gb;
        const uint32_t aoff0 = gdw_off(ra & (R - 1), ca, S.atoms_a), astep = (uint32_t)(rsa / 4) * S.atoms_a * 512;
        const uint32_t boff0 = gdw_off(rb & (R - 1), cb, S.atoms_b), bstep = (uint32_t)(rsb / 4) * S.atoms_b * 512;
        for (int g = 0; g < nst; ++g) {
            const int s = g % S.stages;
            mbar_wait(&bars->landed[s], (g / S.stages) & 1);
            const uint32_t a_hi = sb + s * S.stage, a_lo = a_hi + S.a_half, mk = a_lo + S.a_half;
            const uint32_t b_hi = mk + S.a_half, b_lo = b_hi + S.b_half;
            uint32_t o = aoff0;
            for (int r = ra; r < R; r += rsa, o += astep) {
                const float4 d = lds128(a_hi + o), m = lds128(mk + o);
                const float4 q = make_float4(m.x > 0.f ? d.x : 0.f, m.y > 0.f ? d.y : 0.f, m.z > 0.f ? d.z : 0.f,
                                             m.w > 0.f ? d.w : 0.f);
                float4 hi, lo;
                split4(q, hi, lo);
                sts128(a_hi + o, hi);
                sts128(a_lo + o, lo);
            }
            o = boff0;
            for (int r = rb; r < R; r += rsb, o += bstep) {
                float4 hi, lo;
                split4(lds128(b_hi + o), hi, lo);
                sts128(b_hi + o, hi);
                sts128(b_lo + o, lo);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->full[s]);
        }
    } else if (warp == gdw::MMA_WARP) {
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32_mn(MA, S.N);
            int g = 0;
            for (int p = 0; p < nper; ++p) {
                const int a = p & 1, u = p >> 1;
                if (u >= 1) mbar_wait(&bars->accempty[a], (u - 1) & 1);
                fence_after();
                const uint32_t d = bars->tmem + a * S.N;
                const int g_end = min(nst, (p + 1) * PST);
                for (bool first = true; g < g_end; ++g, first = false) {
                    const int s = g % S.stages;
                    mbar_wait(&bars->full[s], (g / S.stages) & 1);
                    fence_after();
                    const uint32_t a_hi = sb + s * S.stage, a_lo = a_hi + S.a_half;
                    const uint32_t b_hi = a_lo + 2 * S.a_half, b_lo = b_hi + S.b_half;
#pragma unroll
                    for (int kk = 0; kk < R / 8; ++kk) {
                        const uint32_t ao = 2 * kk * S.atoms_a * 512, bo = 2 * kk * S.atoms_b * 512;
                        const uint64_t ah = sdesc_mn(a_hi + ao, 512, S.atoms_a * 512, 1);
                        const uint64_t al = sdesc_mn(a_lo + ao, 512, S.atoms_a * 512, 1);
                        const uint64_t bh = sdesc_mn(b_hi + bo, 512, S.atoms_b * 512, 1);
                        const uint64_t bl = sdesc_mn(b_lo + bo, 512, S.atoms_b * 512, 1);
                        mma_tf32(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                        mma_tf32(d, ah, bl, idesc, 1u);
                        mma_tf32(d, al, bh, idesc, 1u);
                    }
                    commit(&bars->empty[s]);
                }
                commit(&bars->accfull[a]);
            }
        }
        __syncwarp();
    } else {
        // promotion: warp q reads TMEM lane quarter q; accumulator row m sits
        // in lane 32 q + t with m = 32 q + t (M = 128) or m = 16 q + t, t < 16
        // (M = 64).  Each slot element is only ever updated by one thread, in
        // period order: the fp32 sum sequence is fixed.
        const int q = warp & 3;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const int m = MA == 128 ? 32 * q + lane : 16 * q + lane;
        const bool mok = (MA == 128 || lane < 16) && m < hp;
        float* slot = slots + (size_t)blockIdx.x * S.N * MA;   // [N][MA]
        for (int p = 0; p < nper; ++p) {
            const int a = p & 1, u = p >> 1;
            mbar_wait(&bars->accfull[a], u & 1);
            fence_after();
            for (int c0 = 0; c0 < fp; c0 += 8) {
                float v[8];
                tmem_ld8(bars->tmem + lane_off + a * S.N + c0, v);
                tmem_wait_ld();
                if (mok) {
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        if (c0 + t < fp) atomicAdd(slot + (size_t)(c0 + t) * MA + m, v[t]);
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->accempty[a]);
        }
    }
    fence_before();
    __syncthreads();
    if (warp == gdw::MMA_WARP) tmem_dealloc(bars->tmem, S.tmem_cols);
}

// gw[f][h] += sum_cta slot[cta][f][h]   (fp64, fixed order: one warp per
// output, lane l sums slots l, l + 32, ... in order, then a fixed butterfly)
__global__ void gdw_reduce_kernel(int nct, int ma, int n, int fp, int hp, const float* __restrict__ slots,
                                  double* __restrict__ gw) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= (int64_t)fp * hp) return;
    const int f = (int)(i / hp), h = (int)(i % hp);
    double s = 0.0;
    for (int c = lane; c < nct; c += 32) s += (double)__ldg(slots + ((size_t)c * n + f) * ma + h);
    s = warp_sum(s);
    if (lane == 0) gw[i] += s;
}

size_t gcn_dw_tc_workspace(int fp, int hp) {
    if (hp > 128 || fp > 128) return 0;
    const GdwShape S = gdw_shape(hp <= 64 ? 64 : 128, fp);
    return (size_t)num_sms() * S.N * S.MA * sizeof(float) + 256;
}

// -1 when the shape has no instance (the caller then uses the SIMT path)
int gcn_dw_tc(int32_t n, dgnn_frame s, dgnn_frame dr, dgnn_frame r, int fp, int hp, int skip, double* gw, void* ws,
              size_t ws_bytes, cudaStream_t st) {
    // 4-column group counts must be powers of two dividing the converter
    // thread count (fixed per-thread column groups)
    auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
    if (hp > 128 || fp > 128 || hp % 4 || fp % 4 || !pow2(hp / 4) || !pow2(fp / 4)) return -1;
    const int ma = hp <= 64 ? 64 : 128;
    const int rows_st = (fp <= 32 && ma == 64) ? 64 : 32;
    const GdwShape S = gdw_shape(ma, fp, rows_st);
    if (S.stages < 3) return -1;
    const size_t need = (size_t)num_sms() * S.N * S.MA * sizeof(float);
    if (ws_bytes < need) {
        set_error("gcn_weight_grad (tcgen05): workspace too small");
        return DGNN_EWORKSPACE;
    }
    float* slots = reinterpret_cast<float*>(ws);
    cudaMemsetAsync(slots, 0, need, st);
    const size_t smem = (size_t)S.stages * S.stage + 1024 + 256;
    // always one CTA per SM: the CTA row ranges (and so the fp32 period sums)
    // must not depend on dgnn_set_sm_reserve
    const int grid = num_sms();
    const int off = skip ? fp : 0;
    if (ma == 64 && rows_st == 64) {
        cudaFuncSetAttribute(gcn_dw_tc_kernel<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_launch();
        gcn_dw_tc_kernel<64, 64><<<grid, gdw::THREADS, smem, st>>>(n, fp, hp, off, s, dr, r, slots);
    } else if (ma == 64) {
        cudaFuncSetAttribute(gcn_dw_tc_kernel<64, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_launch();
        gcn_dw_tc_kernel<64, 32><<<grid, gdw::THREADS, smem, st>>>(n, fp, hp, off, s, dr, r, slots);
    } else {
        cudaFuncSetAttribute(gcn_dw_tc_kernel<128, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_launch();
        gcn_dw_tc_kernel<128, 32><<<grid, gdw::THREADS, smem, st>>>(n, fp, hp, off, s, dr, r, slots);
    }
    note_launch();
    gdw_reduce_kernel<<<(unsigned)cdiv((int64_t)fp * hp * 32, 256), 256, 0, st>>>(grid, ma, S.N, fp, hp, slots, gw);
    return launch_status("gcn_weight_grad (tcgen05)");
}

}  // namespace dgnn
