// EGCN-O weight evolution on the device: the GCN weight of
// each layer evolves through an elementwise matrix-LSTM over time
// (`egcn_evolve`, models.py:247-268; `evolve_chain_forward/backward`,
// training.py:466-509).  The chain is elementwise over the (padded) F x H
// weight, sequential over the block's timesteps: one thread per element,
// the whole block's chain in registers, fp64 like the reference.  The
// forward writes every step's weight as the fp32 padded image the GCN
// kernels read, plus (rerun) the per-step cache; the backward consumes the
// per-step weight-gradient seeds dW_t (from the GCN weight-gradient kernel)
// and accumulates the gate / bias gradients of the block (summed from zero
// in descending t, then added, as the reference does) and the carry into
// the previous block.
//
// Padded elements (zero weight, zero gate, zero bias) stay exactly zero:
// z = 0 gives c = 0.5 * 0 + 0.5 * tanh(0) = 0 and W = o * tanh(0) = 0.

#include "common.cuh"

namespace dgnn {
namespace {

__device__ __forceinline__ double dsig(double x) { return 1.0 / (1.0 + exp(-x)); }

// cache layout per step: [w_prev | i | f | o | g | tanh c], each `cnt` doubles
__global__ void evolve_fwd_kernel(int64_t cnt, int32_t steps, const double* __restrict__ gates,
                                  const double* __restrict__ bias, const double* __restrict__ w_in,
                                  double* __restrict__ w_out, float* __restrict__ images,
                                  double* __restrict__ cache) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
        const double gi = gates[e], gf = gates[cnt + e], go = gates[2 * cnt + e], gg = gates[3 * cnt + e];
        const double bi = bias[e], bf = bias[cnt + e], bo = bias[2 * cnt + e], bg = bias[3 * cnt + e];
        double w = w_in[e];
        for (int32_t s = 0; s < steps; ++s) {
            // z = gates * w + bias (models.py:262), no contraction
            const double i = dsig(__dadd_rn(__dmul_rn(gi, w), bi));
            const double f = dsig(__dadd_rn(__dmul_rn(gf, w), bf));
            const double o = dsig(__dadd_rn(__dmul_rn(go, w), bo));
            const double g = tanh(__dadd_rn(__dmul_rn(gg, w), bg));
            const double c = __dadd_rn(__dmul_rn(f, w), __dmul_rn(i, g));
            const double tc = tanh(c);
            const double wn = __dmul_rn(o, tc);
            if (cache) {
                double* cs = cache + (int64_t)s * 6 * cnt;
                cs[e] = w;
                cs[cnt + e] = i;
                cs[2 * cnt + e] = f;
                cs[3 * cnt + e] = o;
                cs[4 * cnt + e] = g;
                cs[5 * cnt + e] = tc;
            }
            images[(int64_t)s * cnt + e] = (float)wn;
            w = wn;
        }
        w_out[e] = w;
    }
}

__global__ void evolve_bwd_kernel(int64_t cnt, int32_t steps, const double* __restrict__ gates,
                                  const double* __restrict__ cache, const double* __restrict__ seeds,
                                  double* __restrict__ dw_carry, double* __restrict__ dgates,
                                  double* __restrict__ dbias) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
        const double gk[4] = {gates[e], gates[cnt + e], gates[2 * cnt + e], gates[3 * cnt + e]};
        double dg[4] = {0.0, 0.0, 0.0, 0.0}, db[4] = {0.0, 0.0, 0.0, 0.0};
        double carry = dw_carry[e];
        for (int32_t s = steps - 1; s >= 0; --s) {
            const double* cs = cache + (int64_t)s * 6 * cnt;
            const double wp = cs[e], i = cs[cnt + e], f = cs[2 * cnt + e], o = cs[3 * cnt + e];
            const double g = cs[4 * cnt + e], tc = cs[5 * cnt + e];
            const double dwn = seeds ? __dadd_rn(carry, seeds[(int64_t)s * cnt + e]) : carry;
            const double dout = __dmul_rn(dwn, tc);
            const double dc = __dmul_rn(__dmul_rn(dwn, o), __dadd_rn(1.0, -__dmul_rn(tc, tc)));
            const double df = __dmul_rn(dc, wp), di = __dmul_rn(dc, g), dgg = __dmul_rn(dc, i);
            double dwp = __dmul_rn(dc, f);
            const double dz[4] = {__dmul_rn(__dmul_rn(di, i), __dadd_rn(1.0, -i)),
                                  __dmul_rn(__dmul_rn(df, f), __dadd_rn(1.0, -f)),
                                  __dmul_rn(__dmul_rn(dout, o), __dadd_rn(1.0, -o)),
                                  __dmul_rn(dgg, __dadd_rn(1.0, -__dmul_rn(g, g)))};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                dg[k] = __dadd_rn(dg[k], __dmul_rn(dz[k], wp));
                db[k] = __dadd_rn(db[k], dz[k]);
                dwp = __dadd_rn(dwp, __dmul_rn(dz[k], gk[k]));
            }
            carry = dwp;
        }
        dw_carry[e] = carry;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            dgates[k * cnt + e] += dg[k];
            dbias[k * cnt + e] += db[k];
        }
    }
}

__global__ void scatter_f64_kernel(int64_t n, const double* __restrict__ p, const int64_t* __restrict__ pos,
                                   double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[pos[i]] = p[i];
}

int grid_for(int64_t items) {
    int64_t g = cdiv(items, 128);
    return (int)(g < 1 ? 1 : (g > 4LL * num_sms() ? 4LL * num_sms() : g));
}

}  // namespace
}  // namespace dgnn

extern "C" {

int dgnn_evolve_forward(int64_t cnt, int32_t steps, const double* gates, const double* bias, const double* w_in,
                        double* w_out, float* images, double* cache, void* stream) {
    using namespace dgnn;
    DGNN_CHECK_ARG(cnt >= 0 && steps >= 0, "negative size");
    if (!cnt) return DGNN_OK;
    note_launch();
    evolve_fwd_kernel<<<grid_for(cnt), 128, 0, as_stream(stream)>>>(cnt, steps, gates, bias, w_in, w_out, images,
                                                                    cache);
    return launch_status("dgnn_evolve_forward");
}

int dgnn_scatter_f64(int64_t n, const double* p, const int64_t* pos, double* out, void* stream) {
    using namespace dgnn;
    if (n == 0) return DGNN_OK;
    note_launch();
    scatter_f64_kernel<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(n, p, pos, out);
    return launch_status("dgnn_scatter_f64");
}

int dgnn_evolve_backward(int64_t cnt, int32_t steps, const double* gates, const double* cache, const double* seeds,
                         double* dw_carry, double* dgates, double* dbias, void* stream) {
    using namespace dgnn;
    DGNN_CHECK_ARG(cnt >= 0 && steps >= 0, "negative size");
    if (!cnt) return DGNN_OK;
    note_launch();
    evolve_bwd_kernel<<<grid_for(cnt), 128, 0, as_stream(stream)>>>(cnt, steps, gates, cache, seeds, dw_carry,
                                                                    dgates, dbias);
    return launch_status("dgnn_evolve_backward");
}

}  // extern "C"
