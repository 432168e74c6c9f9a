// refine.cu -- continuous refinement of the discrete stereo labelling (NEXT-2,
// SURVEY 8(f)): the non-convex primal-dual method of Sec. 2.4 with
// the two-slope data approximation of Sec. 3.1, in float32.
//
//   u+ = prox_{tau D~}(u - tau A^T (p - q))            (Eq. cont_iterates, P:306-311,
//   q+ = prox_{tau R_-^*}(q + tau A u)                   grad A of P:350-355, d = 1)
//   p+ = prox_{sigma R_+^*}(p + sigma A(2 u+ - u))
//   prox of (w r_{a,b})^*: Eq. pprox; r = r_{eps,delta} - r_{0,C+delta-eps delta}
//   (Eq. r-decompose); data prox P:431-440; warping P:441.
// Readings R24-R28 as the oracle (oracle/refine.py).
//
// Per pixel state (double [H][W] each): u, p_h, p_v, q_h, q_v (two buffers
// each: every iteration reads one and writes the other, so no thread reads a
// value another thread of the same launch updates), u0 (expansion point), s1,
// s2 (slopes); edge arrays are indexed by the edge's first pixel.  An
// iteration is ONE stencil kernel, one thread per pixel (the dual step's
// neighbouring u+ are recomputed redundantly instead of a second launch); the
// state (104 B/pixel, 48 MB at C2) stays L2-resident across iterations.  A
// warp's `iters` iterations are captured once into a CUDA graph per (frame,
// parameters) and replayed.
#include <cmath>
#include <cstring>

#include "ctx.cuh"

namespace dmm {

namespace {

constexpr int kRX = 32, kRY = 8;
// u (buffers 0, 1), u0 (expansion point), s1, s2, then per buffer b: ph, pv, qh, qv at 5 + 4b
constexpr int kRefArrays = 13;
using real = double;             // float64, the oracle's precision

struct RefArgs {
    real* rf;            // kRefArrays x [H][W]
    const uint8_t* D;    // [H][W][KP]
    const uint8_t* labels;
    int W, H, K, KP;
    real wh, wv, eps, delta, C, h, tau, sigma;
};

__device__ __forceinline__ real* arr(const RefArgs& a, int k) { return a.rf + (size_t)k * a.W * a.H; }

// D at a real label (reading R26): linear interpolation, label clamped to [0, K-1]
__device__ __forceinline__ real d_interp(const uint8_t* Dp, int K, real u) {
    const real uc = fmin(fmax(u, 0.0), (real)(K - 1));
    const int k0 = min((int)floor(uc), K - 1);
    const int k1 = min(k0 + 1, K - 1);
    const real f = uc - (real)k0;
    return (1.0 - f) * (real)Dp[k0] + f * (real)Dp[k1];
}

// prox of step * (w r_{a,b})^* (Eq. pprox)
__device__ __forceinline__ real prox_conj(real t, real w, real a, real b, real step) {
    const real aw = a * w, at = fabs(t);
    const real tp = at <= aw ? t : copysign(fmax(aw, at - b * step), t);
    return fmin(fmax(tp, -w), w);
}

__device__ __forceinline__ real r_dc(real t, real eps, real delta, real C) {
    const real at = fabs(t);
    const real bp = C + delta - eps * delta;
    const real rp = at <= delta ? eps * at : at - delta * (1.0 - eps);
    const real rm = at <= bp ? 0.0 : at - bp;
    return rp - rm;
}

__global__ void refine_init_kernel(RefArgs a) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t i = (size_t)y * a.W + x;
    arr(a, 0)[i] = (real)a.labels[i];
    for (int k = 5; k < kRefArrays; ++k) arr(a, k)[i] = 0.0;
}

// a new expansion point: u0 = u, two-slope approximation (R24)
__global__ void refine_warp_kernel(RefArgs a) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t i = (size_t)y * a.W + x;
    const real u0 = arr(a, 0)[i];
    const uint8_t* Dp = a.D + i * a.KP;
    const real dc = d_interp(Dp, a.K, u0);
    real s1 = (dc - d_interp(Dp, a.K, u0 - a.h)) / a.h;
    real s2 = (d_interp(Dp, a.K, u0 + a.h) - dc) / a.h;
    if (s2 < s1) { const real m = 0.5 * (s1 + s2); s1 = m; s2 = m; }
    arr(a, 2)[i] = u0;
    arr(a, 3)[i] = s1;
    arr(a, 4)[i] = s2;
}

// u+ at pixel j = (jy, jx): prox_{tau D~}(u - tau A^T (p - q)): the two-slope
// data term of stereo (R25; slots 3/4 = s1, s2) or, QUAD, the
// quadratic of flow (Eq. 19/20, R34; slots 3/4 = L, Q)
template <bool QUAD>
__device__ __forceinline__ real primal_u(const RefArgs& a, const real* u, const real* ph, const real* pv,
                                         const real* qh, const real* qv, int jx, int jy) {
    const int W = a.W, H = a.H;
    const size_t j = (size_t)jy * W + jx;
    real div = 0.0;
    if (jx + 1 < W) div += ph[j] - qh[j];
    if (jx > 0) div -= ph[j - 1] - qh[j - 1];
    if (jy + 1 < H) div += pv[j] - qv[j];
    if (jy > 0) div -= pv[j - W] - qv[j - W];
    const real uh = u[j] - a.tau * div;
    const real u0 = arr(a, 2)[j], s1 = arr(a, 3)[j], s2 = arr(a, 4)[j];
    real v;
    if constexpr (QUAD)
        v = (uh + a.tau * (s2 * u0 - s1)) / (1.0 + a.tau * s2);
    else
        v = uh > u0 + a.tau * s2 ? uh - a.tau * s2 : (uh < u0 + a.tau * s1 ? uh - a.tau * s1 : u0);
    return fmin(fmax(v, u0 - a.h), u0 + a.h);
}

// One whole iteration (Eq. cont_iterates) in one kernel: the thread of pixel
// i computes u+ at i and at its right / down neighbours (the dual step of the
// pixel's own edges needs them: a 3-point redundant primal instead of a second
// launch), then q+ (from u) and p+ (from 2u+ - u) of its own edges.  Reads
// buffer cur, writes buffer 1 - cur (u, q) and p in place (each edge owned by
// one pixel, read by no other thread of this launch).
template <bool QUAD>
__global__ void refine_iter_kernel(RefArgs a, int cur) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const int W = a.W, H = a.H;
    const size_t i = (size_t)y * W + x;
    const real* u = arr(a, cur);
    real* un = arr(a, 1 - cur);
    const int b0 = 5 + 4 * cur, b1 = 5 + 4 * (1 - cur);
    const real* ph = arr(a, b0);
    const real* pv = arr(a, b0 + 1);
    const real* qh = arr(a, b0 + 2);
    const real* qv = arr(a, b0 + 3);
    const real ui = u[i];
    const real uni = primal_u<QUAD>(a, u, ph, pv, qh, qv, x, y);
    const real bp = a.C + a.delta - a.eps * a.delta;
    const real bi = 2.0 * uni - ui;
    if (x + 1 < W) {
        const real unr = primal_u<QUAD>(a, u, ph, pv, qh, qv, x + 1, y);
        const real ur = u[i + 1];
        arr(a, b1 + 2)[i] = prox_conj(qh[i] + a.tau * (ui - ur), a.wh, 0.0, bp, a.tau);       // q+ = prox(q + tau A u)
        arr(a, b1)[i] = prox_conj(ph[i] + a.sigma * (bi - (2.0 * unr - ur)), a.wh, a.eps, a.delta, a.sigma);
    }
    if (y + 1 < H) {
        const real und = primal_u<QUAD>(a, u, ph, pv, qh, qv, x, y + 1);
        const real ud = u[i + W];
        arr(a, b1 + 3)[i] = prox_conj(qv[i] + a.tau * (ui - ud), a.wv, 0.0, bp, a.tau);
        arr(a, b1 + 1)[i] = prox_conj(pv[i] + a.sigma * (bi - (2.0 * und - ud)), a.wv, a.eps, a.delta, a.sigma);
    }
    un[i] = uni;
}

__global__ void refine_swap_kernel(RefArgs a) {     // odd iteration count: the state back to buffer 0
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t i = (size_t)y * a.W + x;
    arr(a, 0)[i] = arr(a, 1)[i];
    for (int k = 0; k < 4; ++k) arr(a, 5 + k)[i] = arr(a, 9 + k)[i];
}

// output (disparity units) and the energy E(u) = D(u) + R(Au), double accumulation
__global__ void refine_out_kernel(RefArgs a, real d_min, float* out, double* energy) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    double e = 0.0;
    if (x < a.W && y < a.H) {
        const int W = a.W;
        const size_t i = (size_t)y * W + x;
        const real* u = arr(a, 0);
        const real ui = u[i];
        if (out) out[i] = (float)(d_min + ui);
        e = d_interp(a.D + i * a.KP, a.K, ui);
        if (x + 1 < W) e += a.wh * r_dc(ui - u[i + 1], a.eps, a.delta, a.C);
        if (y + 1 < a.H) e += a.wv * r_dc(ui - u[i + W], a.eps, a.delta, a.C);
    }
    for (int d = 16; d > 0; d >>= 1) e += __shfl_down_sync(0xffffffffu, e, d);
    __shared__ double part[kRX * kRY / 32];
    const int t = threadIdx.y * kRX + threadIdx.x;
    if ((t & 31) == 0) part[t >> 5] = e;
    __syncthreads();
    if (t == 0 && energy) {
        double s = 0.0;
        for (int k = 0; k < kRX * kRY / 32; ++k) s += part[k];
        atomicAdd(energy, s);
    }
}

// ------------------------------------------------------------- optical flow
// D at a real displacement (reading R35): bilinear over the census Hamming
// costs of the four surrounding integer displacements (oob outside the image),
// in the oracle's operation order.
struct FlowArgs {
    const uint32_t* c1;
    const uint32_t* c2;
    int W, H;
    real oob;
};

__device__ __forceinline__ real flow_cost_int(const FlowArgs& f, int x, int y, long long a, long long b) {
    const long long xs = x + a, ys = y + b;
    if (xs < 0 || xs >= f.W || ys < 0 || ys >= f.H) return f.oob;
    return (real)__popc(f.c1[(size_t)y * f.W + x] ^ f.c2[(size_t)ys * f.W + xs]);
}

__device__ __forceinline__ real flow_cost_bilinear(const FlowArgs& f, int x, int y, real u1, real u2) {
    const real a0 = floor(u1), b0 = floor(u2);
    const real fx = u1 - a0, fy = u2 - b0;
    const long long ia = (long long)a0, ib = (long long)b0;
    const real d00 = flow_cost_int(f, x, y, ia, ib), d10 = flow_cost_int(f, x, y, ia + 1, ib);
    const real d01 = flow_cost_int(f, x, y, ia, ib + 1), d11 = flow_cost_int(f, x, y, ia + 1, ib + 1);
    return ((1.0 - fx) * (1.0 - fy) * d00 + fx * (1.0 - fy) * d10) + ((1.0 - fx) * fy * d01 + fx * fy * d11);
}

// the layers' labels -> displacements; duals of both components 0
__global__ void flow_init_kernel(RefArgs a1, RefArgs a2, real u1_min, real u2_min) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a1.W || y >= a1.H) return;
    const size_t i = (size_t)y * a1.W + x;
    arr(a1, 0)[i] = u1_min + (real)a1.labels[i];
    arr(a2, 0)[i] = u2_min + (real)a2.labels[i];
    for (int k = 5; k < kRefArrays; ++k) { arr(a1, k)[i] = 0.0; arr(a2, k)[i] = 0.0; }
}

// the quadratic model of Eq. 19 at the current (u1, u2) (readings R34, R36):
// u0 -> slot 2, L -> slot 3, Q (PSD part) -> slot 4 of each component
__global__ void flow_warp_kernel(RefArgs a1, RefArgs a2, FlowArgs f) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a1.W || y >= a1.H) return;
    const size_t i = (size_t)y * a1.W + x;
    const real u1 = arr(a1, 0)[i], u2 = arr(a2, 0)[i], h = a1.h;
    const real d0 = flow_cost_bilinear(f, x, y, u1, u2);
    const real dp1 = flow_cost_bilinear(f, x, y, u1 + h, u2), dm1 = flow_cost_bilinear(f, x, y, u1 - h, u2);
    const real dp2 = flow_cost_bilinear(f, x, y, u1, u2 + h), dm2 = flow_cost_bilinear(f, x, y, u1, u2 - h);
    arr(a1, 2)[i] = u1;
    arr(a1, 3)[i] = (dp1 - dm1) / (2.0 * h);
    arr(a1, 4)[i] = fmax((dp1 - 2.0 * d0 + dm1) / (h * h), 0.0);
    arr(a2, 2)[i] = u2;
    arr(a2, 3)[i] = (dp2 - dm2) / (2.0 * h);
    arr(a2, 4)[i] = fmax((dp2 - 2.0 * d0 + dm2) / (h * h), 0.0);
}

__global__ void flow_out_kernel(RefArgs a1, RefArgs a2, FlowArgs f, float* out1, float* out2, double* energy) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    double e = 0.0;
    if (x < a1.W && y < a1.H) {
        const int W = a1.W;
        const size_t i = (size_t)y * W + x;
        const real* u1 = arr(a1, 0);
        const real* u2 = arr(a2, 0);
        if (out1) out1[i] = (float)u1[i];
        if (out2) out2[i] = (float)u2[i];
        e = flow_cost_bilinear(f, x, y, u1[i], u2[i]);
        const real* us[2] = {u1, u2};
        for (int k = 0; k < 2; ++k) {
            if (x + 1 < W) e += a1.wh * r_dc(us[k][i] - us[k][i + 1], a1.eps, a1.delta, a1.C);
            if (y + 1 < a1.H) e += a1.wv * r_dc(us[k][i] - us[k][i + W], a1.eps, a1.delta, a1.C);
        }
    }
    for (int d = 16; d > 0; d >>= 1) e += __shfl_down_sync(0xffffffffu, e, d);
    __shared__ double part[kRX * kRY / 32];
    const int t = threadIdx.y * kRX + threadIdx.x;
    if ((t & 31) == 0) part[t >> 5] = e;
    __syncthreads();
    if (t == 0 && energy) {
        double s = 0.0;
        for (int k = 0; k < kRX * kRY / 32; ++k) s += part[k];
        atomicAdd(energy, s);
    }
}

RefArgs ref_args(dmm_ctx* ctx, int frame, const dmm_refine_params* prm) {
    FramePtrs P = frame_ptrs(ctx->L, frame);
    RefArgs a;
    a.rf = reinterpret_cast<real*>(P.rf);
    a.D = P.D;
    a.labels = P.labels;
    a.W = ctx->L.W; a.H = ctx->L.H; a.K = ctx->K; a.KP = ctx->KP;
    a.wh = (real)ctx->cfg.w_h; a.wv = (real)ctx->cfg.w_v;
    a.eps = prm->eps; a.delta = prm->delta; a.C = prm->C; a.h = prm->h; a.tau = prm->tau; a.sigma = prm->sigma;
    return a;
}

}  // namespace

size_t refine_bytes(int W, int H) { return (size_t)kRefArrays * sizeof(real) * W * H; }

dmm_status refine_run(dmm_ctx* ctx, int frame, const dmm_refine_params* prm, float* out, double* energy_dev,
                      cudaStream_t s) {
    FramePtrs P = frame_ptrs(ctx->L, frame);
    RefArgs a = ref_args(ctx, frame, prm);
    const dim3 grid((a.W + kRX - 1) / kRX, (a.H + kRY - 1) / kRY), blk(kRX, kRY);
    refine_init_kernel<<<grid, blk, 0, s>>>(a);
    ++ctx->launches;
    // one warp = the expansion kernel + `iters` iteration kernels (+ a swap for
    // an odd count, so the state ends in buffer 0).  Captured once per (frame,
    // parameters) into a graph on the context's capture stream, replayed on `s`.
    RefineGraph& g = ctx->rg;
    const bool same = g.exec && g.frame == frame && memcmp(&g.prm, prm, sizeof(*prm)) == 0 && g.rf == P.rf;
    if (!same) {
        if (g.exec) { cudaGraphExecDestroy(g.exec); g.exec = nullptr; }
        if (!g.cap && cudaStreamCreateWithFlags(&g.cap, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_status(ctx, cudaGetLastError(), "refine capture stream");
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamBeginCapture(g.cap, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine capture");
        refine_warp_kernel<<<grid, blk, 0, g.cap>>>(a);
        int cur = 0;
        for (int it = 0; it < prm->iters; ++it) {
            refine_iter_kernel<false><<<grid, blk, 0, g.cap>>>(a, cur);
            cur ^= 1;
        }
        if (cur) refine_swap_kernel<<<grid, blk, 0, g.cap>>>(a);
        e = cudaStreamEndCapture(g.cap, &graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine capture end");
        e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine graph instantiate");
        g.frame = frame;
        g.prm = *prm;
        g.rf = P.rf;
    }
    for (int w = 0; w < prm->warps; ++w) {
        cudaError_t e = cudaGraphLaunch(g.exec, s);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine graph launch");
        ctx->launches += 1 + prm->iters + (prm->iters & 1);
    }
    refine_out_kernel<<<grid, blk, 0, s>>>(a, (real)ctx->cfg.d_min, out, energy_dev);
    ++ctx->launches;
    return cuda_status(ctx, cudaGetLastError(), "refine");
}


// Flow refinement (Sec. 3.2): layer frames `frame` (u1) and `frame + 1` (u2)
// of a flow context; census codes of frame `frame`.
dmm_status refine_flow_run(dmm_ctx* ctx, int frame, double u1_min, double u2_min, const dmm_refine_params* prm,
                           float* out1, float* out2, double* energy_dev, cudaStream_t s) {
    RefArgs a1 = ref_args(ctx, frame, prm), a2 = ref_args(ctx, frame + 1, prm);
    FramePtrs P = frame_ptrs(ctx->L, frame);
    FlowArgs f{P.codes_l, P.codes_r, ctx->L.W, ctx->L.H, (real)ctx->oob};
    const dim3 grid((a1.W + kRX - 1) / kRX, (a1.H + kRY - 1) / kRY), blk(kRX, kRY);
    flow_init_kernel<<<grid, blk, 0, s>>>(a1, a2, u1_min, u2_min);
    ++ctx->launches;
    RefineGraph& g = ctx->rgf;
    const bool same = g.exec && g.frame == frame && memcmp(&g.prm, prm, sizeof(*prm)) == 0 && g.rf == P.rf;
    if (!same) {
        if (g.exec) { cudaGraphExecDestroy(g.exec); g.exec = nullptr; }
        if (!g.cap && cudaStreamCreateWithFlags(&g.cap, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_status(ctx, cudaGetLastError(), "refine capture stream");
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamBeginCapture(g.cap, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine capture");
        flow_warp_kernel<<<grid, blk, 0, g.cap>>>(a1, a2, f);
        int cur = 0;
        for (int it = 0; it < prm->iters; ++it) {
            refine_iter_kernel<true><<<grid, blk, 0, g.cap>>>(a1, cur);
            refine_iter_kernel<true><<<grid, blk, 0, g.cap>>>(a2, cur);
            cur ^= 1;
        }
        if (cur) {
            refine_swap_kernel<<<grid, blk, 0, g.cap>>>(a1);
            refine_swap_kernel<<<grid, blk, 0, g.cap>>>(a2);
        }
        e = cudaStreamEndCapture(g.cap, &graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine capture end");
        e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine graph instantiate");
        g.frame = frame;
        g.prm = *prm;
        g.rf = P.rf;
    }
    for (int w = 0; w < prm->warps; ++w) {
        cudaError_t e = cudaGraphLaunch(g.exec, s);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine graph launch");
        ctx->launches += 1 + 2 * prm->iters + 2 * (prm->iters & 1);
    }
    flow_out_kernel<<<grid, blk, 0, s>>>(a1, a2, f, out1, out2, energy_dev);
    ++ctx->launches;
    return cuda_status(ctx, cudaGetLastError(), "flow refine");
}

void refine_release(dmm_ctx* ctx) {
    for (RefineGraph* g : {&ctx->rg, &ctx->rgf}) {
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->cap) cudaStreamDestroy(g->cap);
        g->exec = nullptr;
        g->cap = nullptr;
    }
}

}  // namespace dmm
