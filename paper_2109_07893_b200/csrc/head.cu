// Link-prediction head, softmax cross-entropy and its gradients (K8), plus
// the optimiser and parameter plumbing (K9).
// Reference: models.py:335-348, training.py:102-126, 698-735, 886-900.
#include "common.cuh"

namespace dgnn {

constexpr int kMaxClasses = 8;

// One warp per pair: logits_c = z[u] . hw[:E, c] + z[v] . hw[E:, c] + hb_c
// (lanes stride the embedding), CE in fp64 from the fp32 logits.
__global__ void __launch_bounds__(256) head_loss_kernel(int64_t npairs, const int32_t* __restrict__ u,
                                                        const int32_t* __restrict__ v,
                                                        const int32_t* __restrict__ y, dgnn_frame z, int ep,
                                                        int C, const float* __restrict__ hw,
                                                        const float* __restrict__ hb, double scale,
                                                        double* __restrict__ loss_pp, double* __restrict__ dlogits) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = warp; p < npairs; p += nwarps) {
        const float* zu = frame_row<const float>(z, u[p]);
        const float* zv = frame_row<const float>(z, v[p]);
        float lg[kMaxClasses];
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c) lg[c] = 0.f;
        for (int k = lane; k < ep; k += 32) {
            const float a = zu[k], b = zv[k];
#pragma unroll
            for (int c = 0; c < kMaxClasses; ++c)
                if (c < C) lg[c] += a * hw[k * C + c] + b * hw[(ep + k) * C + c];
        }
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c) lg[c] = warp_sum(lg[c]);
        if (lane == 0) {
            double l[kMaxClasses];
            double mx = -1e300;
            for (int c = 0; c < C; ++c) {
                l[c] = (double)(lg[c] + hb[c]);
                mx = l[c] > mx ? l[c] : mx;
            }
            double se = 0.0;
            for (int c = 0; c < C; ++c) se += exp(l[c] - mx);
            const double lz = log(se);
            const int lab = y[p];
            loss_pp[p] = -((l[lab] - mx) - lz);
            if (dlogits) {
                for (int c = 0; c < C; ++c) {
                    const double pr = exp((l[c] - mx) - lz);
                    dlogits[p * C + c] = (pr - (c == lab ? 1.0 : 0.0)) * scale;
                }
            }
        }
    }
}

// Prediction accuracy (training.py:189-197): first-index argmax of the logits.
__global__ void __launch_bounds__(256) head_predict_kernel(int64_t npairs, const int32_t* __restrict__ u,
                                                           const int32_t* __restrict__ v,
                                                           const int32_t* __restrict__ y, dgnn_frame z, int ep,
                                                           int C, const float* __restrict__ hw,
                                                           const float* __restrict__ hb,
                                                           unsigned long long* correct) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = warp; p < npairs; p += nwarps) {
        const float* zu = frame_row<const float>(z, u[p]);
        const float* zv = frame_row<const float>(z, v[p]);
        float lg[kMaxClasses];
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c) lg[c] = 0.f;
        for (int k = lane; k < ep; k += 32) {
            const float a = zu[k], b = zv[k];
#pragma unroll
            for (int c = 0; c < kMaxClasses; ++c)
                if (c < C) lg[c] += a * hw[k * C + c] + b * hw[(ep + k) * C + c];
        }
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c) lg[c] = warp_sum(lg[c]);
        if (lane == 0) {
            int best = 0;
            float bv = lg[0] + hb[0];
            for (int c = 1; c < C; ++c) {
                const float x = lg[c] + hb[c];
                if (x > bv) { bv = x; best = c; }
            }
            if (best == y[p]) atomicAdd(correct, 1ull);
        }
    }
}

// Head parameter gradient partials: rows 0..2ep-1 of cat^T dlogits, row 2ep = colsum.
// CTA = chunk of pairs; thread t owns output row k = t (k <= 2ep) for all classes.
__global__ void __launch_bounds__(256) head_grad_partial_kernel(int64_t npairs, const int32_t* __restrict__ u,
                                                                const int32_t* __restrict__ v, dgnn_frame z,
                                                                int ep, int C, const double* __restrict__ dl,
                                                                int64_t per, double* __restrict__ part) {
    const int64_t p0 = blockIdx.x * per, p1 = min(npairs, p0 + per);
    const int rows = 2 * ep + 1;
    for (int k = threadIdx.x; k < rows; k += blockDim.x) {
        double acc[kMaxClasses];
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c) acc[c] = 0.0;
        for (int64_t p = p0; p < p1; ++p) {
            double a;
            if (k < ep) a = frame_row<const float>(z, u[p])[k];
            else if (k < 2 * ep) a = frame_row<const float>(z, v[p])[k - ep];
            else a = 1.0;
#pragma unroll
            for (int c = 0; c < kMaxClasses; ++c)
                if (c < C) acc[c] += a * dl[p * C + c];
        }
        for (int c = 0; c < C; ++c) part[((int64_t)blockIdx.x * rows + k) * C + c] = acc[c];
    }
}

__global__ void head_grad_reduce_kernel(int nchunks, int ep, int C, const double* __restrict__ part,
                                        double* __restrict__ ghw, double* __restrict__ ghb) {
    const int rows = 2 * ep + 1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * C) return;
    const int k = i / C, c = i % C;
    double s = 0.0;
    for (int b = 0; b < nchunks; ++b) s += part[((int64_t)b * rows + k) * C + c];
    if (k < 2 * ep) ghw[k * C + c] += s;
    else ghb[c] += s;
}

// dz[x][k] = sum_{slot s of x} sum_c dl[s/2][c] hw[side(s)*ep + k][c]; group of ep/4 lanes per vertex.
// lanes per vertex: GL over every vertex, GLA over an active-vertex list
// (scripts/head_probe.sh)
#ifndef DGNN_HS_GL
#define DGNN_HS_GL 8
#endif
#ifndef DGNN_HS_GLA
#define DGNN_HS_GLA 4
#endif
// threshold (incident slots) above which a vertex is summed by its whole warp
#ifndef DGNN_HS_HUB
#define DGNN_HS_HUB 64
#endif
constexpr int HS_HUB = DGNN_HS_HUB;

// sacc[side][c] += dl[p][c] over the incidence slots e = e, e + stride, ...
// below e1, in slot order; U slots in flight (slot -> dlogit loads issued
// together); predicated adds keep sacc in registers
template <int CM, int U>
__device__ __forceinline__ void hs_fold(int e, int e1, int stride, const int32_t* __restrict__ slot,
                                        const double* __restrict__ dl, int C, double* sacc) {
    for (; e + (U - 1) * stride < e1; e += U * stride) {
        int sl[U];
#pragma unroll
        for (int q = 0; q < U; ++q) sl[q] = slot[e + q * stride];
        double d[U][CM];
#pragma unroll
        for (int q = 0; q < U; ++q)
#pragma unroll
            for (int c = 0; c < CM; ++c) d[q][c] = c < C ? dl[(int64_t)(sl[q] >> 1) * C + c] : 0.0;
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const bool side = sl[q] & 1;
#pragma unroll
            for (int c = 0; c < CM; ++c)
                if (c < C) {
                    if (side) sacc[CM + c] += d[q][c];
                    else sacc[c] += d[q][c];
                }
        }
    }
    for (; e < e1; e += stride) {
        const int sl = slot[e];
        const bool side = sl & 1;
#pragma unroll
        for (int c = 0; c < CM; ++c)
            if (c < C) {
                const double d = dl[(int64_t)(sl >> 1) * C + c];
                if (side) sacc[CM + c] += d;
                else sacc[c] += d;
            }
    }
}

template <int EP, int CC, int GL>   // CC: classes (compile time), 0: runtime C <= kMaxClasses
__global__ void __launch_bounds__(256) head_scatter_kernel(int32_t n, const int32_t* __restrict__ ptr,
                                                           const int32_t* __restrict__ slot,
                                                           const double* __restrict__ dl,
                                                           const float* __restrict__ hw, int C_rt, dgnn_frame dz,
                                                           int32_t nact, const int32_t* __restrict__ act) {
    // dz[x] = sum over x's incident pair endpoints (p, side) of dl[p] . W_side^T
    //       = S_0[x] . W_u^T + S_1[x] . W_v^T,  S_side[x][c] = sum dl[p][c]:
    // 8 lanes per vertex (4 vertices per warp in flight) sum the 2C fp64
    // dlogits over the incidence list, 8 slots at a time, in a fixed
    // butterfly, then form the E outputs -- no vector work per pair; a
    // vertex with more than HS_HUB incident slots (heavy-tailed graphs) is
    // summed by its whole warp.
    // With `act` (the vertices that have incident pairs, ascending), rows
    // without any are zero-filled by a flat float4 pass and the lane
    // groups visit only the active vertices (same arithmetic per row).
    constexpr int CM = CC ? CC : kMaxClasses;
    constexpr int HS_U = CC ? 4 : 1;                // slots per lane in flight (compile-time classes)
    constexpr int PER = (EP + GL - 1) / GL;         // outputs per lane
    const int C = CC ? CC : C_rt;
    extern __shared__ float hws[];                  // [2*EP][C]
    for (int i = threadIdx.x; i < 2 * EP * C; i += blockDim.x) hws[i] = hw[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, gl = lane & (GL - 1);
    if (act) {
        constexpr int Q = EP / 4;
        const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
        for (int64_t i = tid; i < (int64_t)n * Q; i += nth) {
            const int32_t x = (int32_t)(i / Q);
            if (ptr[x + 1] == ptr[x])
                *reinterpret_cast<float4*>(frame_row<float>(dz, x) + 4 * (int)(i % Q)) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    const int64_t nv = act ? nact : n;
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GL;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / GL;
    const int64_t iters = (nv + ngrp - 1) / ngrp;   // uniform trip count: the shuffles need whole warps
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t xi = grp + it * ngrp;
        const bool ok = xi < nv;
        const int64_t x = ok && act ? act[xi] : xi;
        double sacc[2 * CM];
#pragma unroll
        for (int i = 0; i < 2 * CM; ++i) sacc[i] = 0.0;
        const int e0 = ok ? ptr[x] : 0, e1 = ok ? ptr[x + 1] : 0;
        const bool hub = e1 - e0 > HS_HUB;
        if (ok && !hub) hs_fold<CM, HS_U>(e0 + gl, e1, GL, slot, dl, C, sacc);
#pragma unroll
        for (int i = 0; i < 2 * CM; ++i)
#pragma unroll
            for (int o = GL / 2; o > 0; o >>= 1) sacc[i] += __shfl_xor_sync(0xffffffffu, sacc[i], o);
        // vertices with more than HS_HUB incident slots are summed by the
        // whole warp (32 lanes, fixed butterfly), one at a time, and the
        // owning group takes the sums: a hub costs 1/32 of a serial walk
        // instead of 1/GL, and the same in the all-vertex and active passes
        unsigned hubs = __ballot_sync(0xffffffffu, ok && hub && gl == 0);
        while (hubs) {
            const int src = __ffs(hubs) - 1;
            hubs &= hubs - 1;
            const int h0 = __shfl_sync(0xffffffffu, e0, src), h1 = __shfl_sync(0xffffffffu, e1, src);
            double hs[2 * CM];
#pragma unroll
            for (int i = 0; i < 2 * CM; ++i) hs[i] = 0.0;
            hs_fold<CM, HS_U>(h0 + lane, h1, 32, slot, dl, C, hs);
#pragma unroll
            for (int i = 0; i < 2 * CM; ++i) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) hs[i] += __shfl_xor_sync(0xffffffffu, hs[i], o);
                if (lane / GL == src / GL) sacc[i] = hs[i];
            }
        }
        if (!ok) continue;
        float* out = frame_row<float>(dz, x);
        float v[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int k = gl * PER + j;
            double a = 0.0;
            if (k < EP)
                for (int c = 0; c < C; ++c)
                    a += sacc[c] * (double)hws[k * C + c] + sacc[CM + c] * (double)hws[(EP + k) * C + c];
            v[j] = (float)a;
        }
#pragma unroll
        for (int j = 0; j < PER; j += 4)
            if (gl * PER + j < EP)
                *reinterpret_cast<float4*>(out + gl * PER + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
}

// Adam (training.py:886-900), IEEE-rounded ops in the reference's order.
__global__ void adam_kernel(int64_t n, double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                            double* __restrict__ v, double lr, double b1, double one_m_b1, double b2,
                            double one_m_b2, double bc1, double bc2, double eps) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double gi = g[i];
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(one_m_b1, gi));
    const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(one_m_b2, __dmul_rn(gi, gi)));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, bc1), vh = __ddiv_rn(vi, bc2);
    const double step = __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps));
    p[i] = __dsub_rn(p[i], step);
}

__global__ void params_to_device_kernel(int64_t n, const double* __restrict__ p, const int64_t* __restrict__ pos0,
                                        const int64_t* __restrict__ pos1, float* __restrict__ w) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float f = (float)p[i];
    w[pos0[i]] = f;
    if (pos1 && pos1[i] >= 0) w[pos1[i]] = f;
}

__global__ void grads_gather_kernel(int64_t n, const double* __restrict__ gp, const int64_t* __restrict__ pos0,
                                    double* __restrict__ g) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) g[i] = gp[pos0[i]];
}

template <int EP>
int head_scatter_t(int32_t n, const int32_t* ptr, const int32_t* slot, const double* dl, const float* hw, int C,
                   dgnn_frame dz, cudaStream_t st, int32_t nact = 0, const int32_t* act = nullptr) {
    if (C > kMaxClasses) {
        set_error("head_scatter: %d classes exceed %d", C, kMaxClasses);
        return DGNN_EUNSUPPORTED;
    }
    int64_t blocks = cdiv(n, 32);
#ifndef DGNN_HS_BLK
#define DGNN_HS_BLK 16
#endif
    blocks = blocks < 1 ? 1 : (blocks > DGNN_HS_BLK * num_sms() ? DGNN_HS_BLK * num_sms() : blocks);
    ::dgnn::note_launch();
    const size_t sm = (size_t)2 * EP * C * sizeof(float);
    if (act) {
        if (C == 2)
            head_scatter_kernel<EP, 2, DGNN_HS_GLA><<<(unsigned)blocks, 256, sm, st>>>(n, ptr, slot, dl, hw, C, dz, nact, act);
        else
            head_scatter_kernel<EP, 0, DGNN_HS_GLA><<<(unsigned)blocks, 256, sm, st>>>(n, ptr, slot, dl, hw, C, dz, nact, act);
    } else if (C == 2) {
        head_scatter_kernel<EP, 2, DGNN_HS_GL><<<(unsigned)blocks, 256, sm, st>>>(n, ptr, slot, dl, hw, C, dz, 0, nullptr);
    } else {
        head_scatter_kernel<EP, 0, DGNN_HS_GL><<<(unsigned)blocks, 256, sm, st>>>(n, ptr, slot, dl, hw, C, dz, 0, nullptr);
    }
    return launch_status("head_scatter");
}


// Fused head loss + head-parameter gradient (one pass over the labelled
// pairs, training.py:698-735).  LP = EP / D lanes per pair (D embedding
// dims each), 32 / LP pairs per warp in flight.  Logits are reduced over the
// group in a fixed butterfly and taken from the group leader, which does
// the fp64 softmax CE, writes loss_pp and dlogits (the scatter kernel reads
// them) and broadcasts dl to its group; every lane folds a * dl into fp64
// accumulators of its D dims (u and v side).  Pairs are assigned statically
// (fixed grid), groups / warps / CTAs are combined in fixed order and the
// per-CTA partials are reduced by head_lg_reduce_kernel: deterministic.
// two CTAs per SM (<= 128 registers): the pair loop is a chain of dependent
// gathers, so resident warps are what hides it
#ifndef DGNN_HEAD_CPS
#define DGNN_HEAD_CPS 2
#endif
// embedding dims per lane: 8 (4 removes the register spills at two CTAs per
// SM but measured slower: 63 -> 80 us at configs[2], scripts/head_lg_time.py)
#ifndef DGNN_HEAD_DIMS
#define DGNN_HEAD_DIMS 8
#endif
static int head_ctas() { return DGNN_HEAD_CPS * num_sms(); }

template <int EP>
__global__ void __launch_bounds__(256, DGNN_HEAD_CPS) head_loss_grad_kernel(int64_t npairs, const int32_t* __restrict__ u,
                                                             const int32_t* __restrict__ v,
                                                             const int32_t* __restrict__ y, dgnn_frame z, int C,
                                                             const float* __restrict__ hw,
                                                             const float* __restrict__ hb, double scale,
                                                             double* __restrict__ loss_pp,
                                                             double* __restrict__ dlogits,
                                                             double* __restrict__ part) {
    constexpr int D = DGNN_HEAD_DIMS;          // embedding dims per lane
    constexpr int LP = EP / D;                 // lanes per pair
    constexpr int ROWS = 2 * EP + 1;           // head.w rows (u side, v side) + bias
    __shared__ float hws[2 * EP * kMaxClasses];
    __shared__ double red[8][ROWS * 2];        // per-warp partials (C <= 2 staged here; see below)
    for (int i = threadIdx.x; i < 2 * EP * C; i += blockDim.x) hws[i] = hw[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gl = lane % LP, grp = lane / LP;
    const unsigned gmask = (LP == 32 ? 0xffffffffu : (((1u << LP) - 1u) << (grp * LP)));
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LP;
    const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / LP;
    const int k0 = D * gl;
    double acc_u[D][2], acc_v[D][2], acc_b[2];
#pragma unroll
    for (int j = 0; j < D; ++j) acc_u[j][0] = acc_u[j][1] = acc_v[j][0] = acc_v[j][1] = 0.0;
    acc_b[0] = acc_b[1] = 0.0;
    // the next pair's endpoints are loaded one iteration ahead, so
    // an iteration waits on one gather latency (z rows), not two
    int32_t un = 0, vn = 0;
    if (gid < npairs) {
        un = u[gid];
        vn = v[gid];
    }
    for (int64_t p = gid; p < npairs; p += ngroups) {
        const int32_t uc = un, vc = vn;
        const int lab = gl == 0 ? y[p] : 0;   // issued here, used after the logits
        if (p + ngroups < npairs) {
            un = u[p + ngroups];
            vn = v[p + ngroups];
        }
        const float4* zu = reinterpret_cast<const float4*>(frame_row<const float>(z, uc) + k0);
        const float4* zv = reinterpret_cast<const float4*>(frame_row<const float>(z, vc) + k0);
        float a[D], b[D];
#pragma unroll
        for (int q = 0; q < D / 4; ++q) {
            const float4 aq = zu[q], bq = zv[q];
            a[4 * q] = aq.x, a[4 * q + 1] = aq.y, a[4 * q + 2] = aq.z, a[4 * q + 3] = aq.w;
            b[4 * q] = bq.x, b[4 * q + 1] = bq.y, b[4 * q + 2] = bq.z, b[4 * q + 3] = bq.w;
        }
        float lg[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            float t = 0.f;
            if (c < C) {
#pragma unroll
                for (int j = 0; j < D; ++j) t += a[j] * hws[(k0 + j) * C + c] + b[j] * hws[(EP + k0 + j) * C + c];
            }
#pragma unroll
            for (int o = LP / 2; o > 0; o >>= 1) t += __shfl_xor_sync(gmask, t, o);
            lg[c] = __shfl_sync(gmask, t, grp * LP);   // the leader's value: one rounding for the group
        }
        double dl[2] = {0.0, 0.0};
        if (gl == 0) {
            const double l0 = (double)(lg[0] + hb[0]), l1 = (double)(lg[1] + hb[1]);
            const double mx = l0 > l1 ? l0 : l1;
            const double lz = log(exp(l0 - mx) + exp(l1 - mx));
            loss_pp[p] = -(((lab ? l1 : l0) - mx) - lz);
            dl[0] = (exp((l0 - mx) - lz) - (lab == 0 ? 1.0 : 0.0)) * scale;
            dl[1] = (exp((l1 - mx) - lz) - (lab == 1 ? 1.0 : 0.0)) * scale;
            dlogits[p * 2] = dl[0];
            dlogits[p * 2 + 1] = dl[1];
            acc_b[0] += dl[0];
            acc_b[1] += dl[1];
        }
        dl[0] = __shfl_sync(gmask, dl[0], grp * LP);
        dl[1] = __shfl_sync(gmask, dl[1], grp * LP);
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                acc_u[j][c] += (double)a[j] * dl[c];
                acc_v[j][c] += (double)b[j] * dl[c];
            }
    }
    // groups of a warp -> group 0 (fixed order: group g adds group g + span)
#pragma unroll
    for (int span = 16; span >= LP; span >>= 1) {
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                acc_u[j][c] += __shfl_down_sync(0xffffffffu, acc_u[j][c], span);
                acc_v[j][c] += __shfl_down_sync(0xffffffffu, acc_v[j][c], span);
            }
        acc_b[0] += __shfl_down_sync(0xffffffffu, acc_b[0], span);
        acc_b[1] += __shfl_down_sync(0xffffffffu, acc_b[1], span);
    }
    if (lane < LP) {
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                red[warp][(k0 + j) * 2 + c] = acc_u[j][c];
                red[warp][(EP + k0 + j) * 2 + c] = acc_v[j][c];
            }
        if (lane == 0) {
            red[warp][2 * EP * 2] = acc_b[0];
            red[warp][2 * EP * 2 + 1] = acc_b[1];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ROWS * 2; i += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w][i];
        part[(int64_t)blockIdx.x * ROWS * 2 + i] = t;
    }
}

// ghw[k][c] (k < 2 ep) / ghb[c] += sum over CTAs of part (fixed tree)
__global__ void __launch_bounds__(128) head_lg_reduce_kernel(int nct, int outs, int ep,
                                                             const double* __restrict__ part,
                                                             double* __restrict__ ghw, double* __restrict__ ghb) {
    __shared__ double sh[128];
    const int i = blockIdx.x;   // output index: row k = i / 2, class c = i % 2
    double t = 0.0;
    for (int b = threadIdx.x; b < nct; b += 128) t += part[(int64_t)b * outs + i];
    sh[threadIdx.x] = t;
    __syncthreads();
    for (int o = 64; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int k = i / 2, c = i % 2;
        if (k < 2 * ep) ghw[k * 2 + c] += sh[0];
        else ghb[c] += sh[0];
    }
}

template <int EP>
int head_loss_grad_t(int64_t npairs, const int32_t* u, const int32_t* v, const int32_t* y, dgnn_frame z,
                     const float* hw, const float* hb, double scale, double* loss_pp, double* dlogits, double* ghw,
                     double* ghb, double* part, cudaStream_t st) {
    int64_t blocks = cdiv(npairs, 256 / (EP / DGNN_HEAD_DIMS));
    blocks = blocks > head_ctas() ? head_ctas() : (blocks < 1 ? 1 : blocks);
    note_launch();
    head_loss_grad_kernel<EP><<<(unsigned)blocks, 256, 0, st>>>(npairs, u, v, y, z, 2, hw, hb, scale, loss_pp,
                                                                 dlogits, part);
    const int outs = (2 * EP + 1) * 2;
    note_launch();
    head_lg_reduce_kernel<<<(unsigned)outs, 128, 0, st>>>((int)blocks, outs, EP, part, ghw, ghb);
    return launch_status("head_loss_grad");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

int dgnn_head_loss(int64_t npairs, const int32_t* u, const int32_t* v, const int32_t* y, dgnn_frame z,
                   int32_t ep, int32_t c, const float* hw, const float* hb, double scale, double* loss_pp,
                   int32_t n_partials, double* dlogits, void* stream) {
    DGNN_CHECK_ARG(c >= 2 && c <= kMaxClasses, "head_loss: classes outside [2, 8]");
    DGNN_CHECK_ARG(n_partials >= npairs, "head_loss: per-pair loss buffer too small");
    if (npairs == 0) return DGNN_OK;
    int64_t blocks = cdiv(npairs, 8);
    blocks = blocks > 32 * num_sms() ? 32 * num_sms() : blocks;
    ::dgnn::note_launch();
    head_loss_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(npairs, u, v, y, z, ep, c, hw, hb, scale,
                                                                      loss_pp, dlogits);
    return launch_status("head_loss");
}

int dgnn_head_predict(int64_t npairs, const int32_t* u, const int32_t* v, const int32_t* y, dgnn_frame z,
                      int32_t ep, int32_t c, const float* hw, const float* hb, int64_t* correct, void* stream) {
    DGNN_CHECK_ARG(c >= 2 && c <= kMaxClasses, "head_predict: classes outside [2, 8]");
    if (npairs == 0) return DGNN_OK;
    int64_t blocks = cdiv(npairs, 8);
    blocks = blocks > 32 * num_sms() ? 32 * num_sms() : blocks;
    ::dgnn::note_launch();
    head_predict_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        npairs, u, v, y, z, ep, c, hw, hb, reinterpret_cast<unsigned long long*>(correct));
    return launch_status("head_predict");
}

size_t dgnn_head_grad_workspace(int32_t ep, int32_t c) {
    return (size_t)(4 * num_sms()) * (2 * ep + 1) * c * sizeof(double) + 256;
}

int dgnn_head_grad(int64_t npairs, const int32_t* u, const int32_t* v, dgnn_frame z, int32_t ep, int32_t c,
                   const double* dlogits, double* ghw, double* ghb, void* ws, size_t ws_bytes, void* stream) {
    DGNN_CHECK_ARG(c >= 2 && c <= kMaxClasses, "head_grad: classes outside [2, 8]");
    if (ws_bytes < dgnn_head_grad_workspace(ep, c)) {
        set_error("head_grad: workspace too small");
        return DGNN_EWORKSPACE;
    }
    if (npairs == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    int64_t nch = cdiv(npairs, 256);
    nch = nch > 4 * num_sms() ? 4 * num_sms() : nch;
    const int64_t per = cdiv(npairs, nch);
    nch = cdiv(npairs, per);
    double* part = reinterpret_cast<double*>(ws);
    ::dgnn::note_launch();
    head_grad_partial_kernel<<<(unsigned)nch, 256, 0, st>>>(npairs, u, v, z, ep, c, dlogits, per, part);
    const int outs = (2 * ep + 1) * c;
    ::dgnn::note_launch();
    head_grad_reduce_kernel<<<(unsigned)cdiv(outs, 256), 256, 0, st>>>((int)nch, ep, c, part, ghw, ghb);
    return launch_status("head_grad");
}

int dgnn_head_loss_grad(int64_t npairs, const int32_t* u, const int32_t* v, const int32_t* y, dgnn_frame z,
                        int32_t ep, int32_t c, const float* hw, const float* hb, double scale, double* loss_pp,
                        int32_t n_partials, double* dlogits, double* ghw, double* ghb, void* ws, size_t ws_bytes,
                        void* stream) {
    DGNN_CHECK_ARG(c == 2, "head_loss_grad: the fused kernel serves the 2-class link predictor");
    DGNN_CHECK_ARG(n_partials >= npairs, "head_loss_grad: per-pair loss buffer too small");
    if (ws_bytes < dgnn_head_grad_workspace(ep, c)) {
        set_error("head_loss_grad: workspace too small");
        return DGNN_EWORKSPACE;
    }
    if (npairs == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    double* part = reinterpret_cast<double*>(ws);
    switch (ep) {
        case 16: return head_loss_grad_t<16>(npairs, u, v, y, z, hw, hb, scale, loss_pp, dlogits, ghw, ghb, part, st);
        case 32: return head_loss_grad_t<32>(npairs, u, v, y, z, hw, hb, scale, loss_pp, dlogits, ghw, ghb, part, st);
        case 64: return head_loss_grad_t<64>(npairs, u, v, y, z, hw, hb, scale, loss_pp, dlogits, ghw, ghb, part, st);
        case 128: return head_loss_grad_t<128>(npairs, u, v, y, z, hw, hb, scale, loss_pp, dlogits, ghw, ghb, part, st);
    }
    set_error("head_loss_grad: unsupported width %d", ep);
    return DGNN_EUNSUPPORTED;
}

int dgnn_head_scatter_active(int32_t n, const int32_t* inc_ptr, const int32_t* inc_slot, int32_t n_active,
                             const int32_t* active, const double* dlogits, const float* hw, int32_t ep, int32_t c,
                             dgnn_frame dz, void* stream) {
    DGNN_CHECK_ARG(c >= 1 && c <= kMaxClasses, "head_scatter: classes outside [1, 8]");
    DGNN_CHECK_ARG(n_active >= 0 && (active || n_active == 0), "head_scatter: bad active list");
    if (n == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    const int32_t* act = active ? active : inc_ptr;   // non-null: zero-fill pass on, n_active = 0 visits nothing
    switch (ep) {
        case 16: return head_scatter_t<16>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st, n_active, act);
        case 32: return head_scatter_t<32>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st, n_active, act);
        case 64: return head_scatter_t<64>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st, n_active, act);
        case 128: return head_scatter_t<128>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st, n_active, act);
    }
    set_error("head_scatter: unsupported width %d", ep);
    return DGNN_EUNSUPPORTED;
}

int dgnn_head_scatter(int32_t n, const int32_t* inc_ptr, const int32_t* inc_slot, const double* dlogits,
                      const float* hw, int32_t ep, int32_t c, dgnn_frame dz, void* stream) {
    DGNN_CHECK_ARG(c >= 1 && c <= kMaxClasses, "head_scatter: classes outside [1, 8]");
    if (n == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (ep) {
        case 16: return head_scatter_t<16>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st);
        case 32: return head_scatter_t<32>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st);
        case 64: return head_scatter_t<64>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st);
        case 128: return head_scatter_t<128>(n, inc_ptr, inc_slot, dlogits, hw, c, dz, st);
    }
    set_error("head_scatter: unsupported width %d", ep);
    return DGNN_EUNSUPPORTED;
}

int dgnn_adam(int64_t n, double* p, const double* g, double* m, double* v, double lr, double beta1,
                 double one_m_beta1, double beta2, double one_m_beta2, double bc1, double bc2, double eps,
                 void* stream) {
    if (n == 0) return DGNN_OK;
    ::dgnn::note_launch();
    adam_kernel<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(n, p, g, m, v, lr, beta1, one_m_beta1,
                                                                       beta2, one_m_beta2, bc1, bc2, eps);
    return launch_status("adam");
}

int dgnn_params_to_device(int64_t n, const double* p, const int64_t* pos0, const int64_t* pos1, float* w32,
                          void* stream) {
    if (n == 0) return DGNN_OK;
    ::dgnn::note_launch();
    params_to_device_kernel<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(n, p, pos0, pos1, w32);
    return launch_status("params_to_device");
}

int dgnn_grads_gather(int64_t n, const double* gpad, const int64_t* pos0, double* g, void* stream) {
    if (n == 0) return DGNN_OK;
    ::dgnn::note_launch();
    grads_gather_kernel<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(n, gpad, pos0, g);
    return launch_status("grads_gather");
}

}  // extern "C"
