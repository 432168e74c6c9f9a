// capi.cu -- the extern "C" boundary declared in include/dmm.h: argument
// checks, workspace carving, kernel orchestration of Algorithm 2,
// and error reporting.  No torch types cross this boundary.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dmm.h"
#include "dmm_internal.cuh"

#include "ctx.cuh"

namespace {

constexpr int kPartial = -1;   // iters_done of a DMM_TUNE_DEBUG_STOP_AFTER_H solve

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

bool valid(const dmm_config* c) {
    if (!c) return false;
    if (c->pen_e1 < 0 || c->pen_e2 < c->pen_e1 || c->pen_delta < 0 || c->pen_c < 0 || c->pen_c > (1 << 20) ||
        c->pen_e2 > (1 << 20) || (c->edge_weights != 0 && c->edge_weights != 1))
        return false;
    if (c->minorant < 0 || c->minorant > 1 ||
        (c->minorant == 1 && (c->iter_passes < 1 || c->iter_passes > 64 || c->iter_gshift < 0 || c->iter_gshift > 16)))
        return false;
    const int K = c->d_max - c->d_min + 1;
    // width <= 16384: cost_kernel stages the row's two code rows (8 * W bytes) in
    // shared memory; W * H <= 2^28 keeps every pixel index in int32.
    return c->width >= 1 && c->height >= 1 && c->width <= (1 << 14) && c->height <= (1 << 14) &&
           K >= 1 && K <= 256 && (c->census_radius == 1 || c->census_radius == 2) &&
           c->w_h >= 0 && c->w_v >= 0 && c->w_h <= 255 && c->w_v <= 255 && c->trunc >= 1 &&
           c->frac_bits >= 0 && c->frac_bits <= 8 && c->oob_cost >= -1 && c->oob_cost <= 255 &&
           c->batch >= 1 && c->max_iters >= 1 && c->max_iters <= 1024;
}

// Span bound of every stored K-vector: a Msg
// output spans <= ws*min(T, K-1); f_ = L + D_s + R and D_s + g_ = D_s + L + R
// span <= (2*w*min(T, K-1) + maxD) * 2^F.  Records store u16 offsets.
long long span_bound(const dmm_config* c) {
    const int K = c->d_max - c->d_min + 1;
    const int r = c->census_radius;
    const int bits = (2 * r + 1) * (2 * r + 1) - 1;
    const int oob = c->oob_cost >= 0 ? c->oob_cost : bits / 2;
    const long long maxD = oob > bits ? oob : bits;
    const long long w = c->w_h > c->w_v ? c->w_h : c->w_v;
    const long long T = c->trunc < K - 1 ? c->trunc : (K - 1);
    return (2 * w * T + maxD) << c->frac_bits;
}

// Range check of the packed chain-pair kernels (hm2.cu, hm2_device.cuh): with
// wsT = w*2^F*min(T, K) and S = span_bound, a pass leaves its message
// unnormalised for at most 16 steps (the ring chunk), during which its minimum
// drifts up by <= S per step, so every packed operand lies in
// [-wsT - 1, 16*S + wsT] and every distance-transform candidate (addends are
// clamped to wsT + 1) below 16*S + 2*wsT + 2; 16*S + 3*wsT + 4 <= 16383 (the
// packed "infinity", with 16383 + wsT + 1 <= 32767) keeps all values and
// candidates exact in signed 16 bits.
bool pair_range_ok(const dmm_config* c) {
    const long long K = c->d_max - c->d_min + 1;
    const long long w = c->w_h > c->w_v ? c->w_h : c->w_v;
    const long long T = c->trunc < K ? c->trunc : K;
    const long long wsT = (w << c->frac_bits) * T;
    const int bits = (2 * c->census_radius + 1) * (2 * c->census_radius + 1) - 1;
    const int oob = c->oob_cost >= 0 ? c->oob_cost : bits / 2;
    // D < 128: the packed D unpack zero-fills with sign-replicated bytes
    return 16 * span_bound(c) + 3 * wsT + 4 <= 16383 && oob < 128 && bits < 128;
}

int kp_of(int K) {
    int lpl = 1;
    while (32 * lpl < K) lpl *= 2;
    return 32 * lpl;
}

// Byte offsets of every array inside one frame block; returns the block size.
size_t frame_layout(const dmm_config* c, dmm::FramePtrs* off) {
    const size_t W = c->width, H = c->height, KP = kp_of(c->d_max - c->d_min + 1);
    const size_t px = W * H, cells = px * KP;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
    off->img_l = (uint8_t*)take(px);
    off->img_r = (uint8_t*)take(px);
    off->codes_l = (uint32_t*)take(4 * px);
    off->codes_r = (uint32_t*)take(4 * px);
    off->D = (uint8_t*)take(cells);
    off->fv = (uint8_t*)take(px * (size_t)dmm::rec_bytes((int)KP));
    off->fh = (uint8_t*)take(px * (size_t)dmm::rec_bytes((int)KP));
    off->fwd = (int32_t*)take(4 * cells);
    off->bwd = (int32_t*)take(4 * cells);
    off->fwdo = (int32_t*)take(8 * px);
    off->bwdo = (int32_t*)take(8 * px);
    off->labels = (uint8_t*)take(px);
    off->bounds = (long long*)take(8 * 2 * (size_t)c->max_iters);
    off->energy = (long long*)take(8);
    off->flag = (int32_t*)take(8);
    off->tmap = (uint8_t*)take(dmm::kTmapBytes);
    off->rf = (float*)take(dmm::refine_bytes((int)W, (int)H));
    off->renergy = (double*)take(8);
    if (dmm::gen_mode(c)) {
        off->gfv = (int32_t*)take(4 * cells);
        off->ggh = (int32_t*)take(4 * cells);
        off->gom_h = (uint8_t*)take(px);
        off->gom_v = (uint8_t*)take(px + 256);
    }
    return o;
}

dmm_status cuda_err(dmm_ctx* ctx, cudaError_t e, const char* where) {
    if (e == cudaSuccess) return DMM_OK;
    if (ctx) ctx->err = std::string(where) + ": " + cudaGetErrorString(e);
    return DMM_E_CUDA;
}

dmm_status check_launch(dmm_ctx* ctx, const char* where) {
    return cuda_err(ctx, cudaGetLastError(), where);
}

cudaEvent_t get_event(dmm_ctx* c) {
    if (!c->pool.empty()) { cudaEvent_t e = c->pool.back(); c->pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets one kernel launch with events when profiling is on.
struct Timed {
    dmm_ctx* c; int cls; cudaStream_t s; cudaEvent_t a = nullptr;
    int count;
    Timed(dmm_ctx* c_, int cls_, cudaStream_t s_, int count_ = 1) : c(c_), cls(cls_), s(s_), count(count_) {
        if (c->profiling) { a = get_event(c); cudaEventRecord(a, s); }
    }
    ~Timed() {
        c->launches += count;
        if (a) {
            cudaEvent_t b = get_event(c);
            cudaEventRecord(b, s);
            c->recs.push_back({cls, a, b});
        }
    }
};

// Every entry point that takes a context runs on the context's device and
// restores the caller's current device on return (contexts on
// several devices in one thread).
struct DevGuard {
    int prev = -1;
    bool sw = false;
    explicit DevGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) sw = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DevGuard() {
        if (sw) cudaSetDevice(prev);
    }
};
#define DMM_DEVICE_GUARD(ctx) DevGuard dmm_dev_guard_((ctx)->device)

dmm_status frame_ok(dmm_ctx* ctx, int frame, int n = 1) {
    if (!ctx || frame < 0 || n < 1 || frame + n > ctx->cfg.batch) {
        if (ctx) ctx->err = "frame index out of range";
        return DMM_E_ARG;
    }
    return DMM_OK;
}

}  // namespace

namespace dmm {

dmm_status cuda_status(dmm_ctx* ctx, cudaError_t e, const char* where) { return cuda_err(ctx, e, where); }

// One half-step (vertical = 0: H, 1: V) of iteration t on frames [frame,
// frame+nframes) of layout L (the context's frames, or a shard's band).
dmm_status launch_half_on(dmm_ctx* ctx, const Layout& L, int frame, int nframes, int t, int v, int iterations,
                          int nseg, const int* segx, cudaStream_t s) {
    const int T = ctx->cfg.trunc < ctx->K ? ctx->cfg.trunc : ctx->K;   // T >= K: untruncated
    PassArgs a;
    a.L = L;
    a.frame0 = frame;
    a.fbits = ctx->cfg.frac_bits;
    a.ws = (v ? ctx->cfg.w_v : ctx->cfg.w_h) << ctx->cfg.frac_bits;
    a.wsT = a.ws * T;
    a.T = T;
    a.first = (t == 0 && v == 0);
    a.last = (t == iterations - 1 && v == 1);
    a.bound_slot = 2 * t + v;
    a.nseg = nseg;
    a.segx = segx;
    a.vtma = (&L == &ctx->sh.Lv) ? ctx->sh.vtma : ctx->vtma;
    if (gen_mode(&ctx->cfg)) {
        Timed tm(ctx, 2 + v, s, 0);
        gen_half(ctx, frame, nframes, t, v, iterations, s);
        return check_launch(ctx, "general half step");
    }
    if (ctx->use_pair && ctx->pair_ok) {
        Timed tm(ctx, 2 + v, s, hm2_launches_per_pass(a, v));
        launch_hm2_pass(a, v, nframes, s);
    } else {
        Timed tm(ctx, 2 + v, s, hm_launches_per_pass(a, v, 0));
        launch_hm_pass(a, v, nframes, 0, s);
    }
    return check_launch(ctx, "half step");
}

}  // namespace dmm

namespace {

void launch_half(dmm_ctx* ctx, int frame, int nframes, int t, int v, int iterations, cudaStream_t s) {
    dmm::launch_half_on(ctx, ctx->L, frame, nframes, t, v, iterations, 1, nullptr, s);
}

bool rowcol(const dmm_ctx* ctx) { return ctx->sh.mode == DMM_SHARD_ROWCOL; }

dmm_status not_sharded(dmm_ctx* ctx, const char* what) {
    if (!rowcol(ctx)) return DMM_OK;
    ctx->err = std::string(what) + " is not available on a band-sharded context";
    return DMM_E_STATE;
}

}  // namespace

extern "C" {

size_t dmm_workspace_bytes(const dmm_config* cfg) {
    if (!valid(cfg)) return 0;
    dmm::FramePtrs off;
    return frame_layout(cfg, &off) * (size_t)cfg->batch;
}

dmm_status dmm_create(const dmm_config* cfg, void* workspace, size_t bytes, int device,
                      dmm_ctx** out) {
    if (!out || !valid(cfg) || !workspace || ((uintptr_t)workspace & 255)) return DMM_E_ARG;
    if (dmm::gen_mode(cfg)) {
        // every message / minorant value is bounded by a chain's cost of the
        // optimal labelling plus the same of the other orientation's dual;
        // 4 n (maxD 2^F + 2 w c) < 2^30 keeps all int32 sums exact
        const int bits = (2 * cfg->census_radius + 1) * (2 * cfg->census_radius + 1) - 1;
        const long long maxD = (cfg->oob_cost > bits ? cfg->oob_cost : bits) << cfg->frac_bits;
        const long long w = cfg->w_h > cfg->w_v ? cfg->w_h : cfg->w_v;
        const long long n = cfg->width > cfg->height ? cfg->width : cfg->height;
        const long long cap = (cfg->pen_e1 || cfg->pen_e2 || cfg->pen_delta || cfg->pen_c)
                                  ? cfg->pen_c : ((long long)cfg->trunc << cfg->frac_bits);
        if (4 * n * (maxD + 2 * w * cap) >= (1ll << 30)) return DMM_E_RANGE;
    } else if (span_bound(cfg) > 65535) {
        return DMM_E_RANGE;
    }
    *out = nullptr;
    if (bytes < dmm_workspace_bytes(cfg)) return DMM_E_ARG;
    dmm_ctx* c = new (std::nothrow) dmm_ctx();
    if (!c) return DMM_E_ARG;
    c->cfg = *cfg;
    c->K = cfg->d_max - cfg->d_min + 1;
    c->KP = kp_of(c->K);
    c->device = device;
    c->oob = cfg->oob_cost >= 0 ? cfg->oob_cost
                                : ((2 * cfg->census_radius + 1) * (2 * cfg->census_radius + 1) - 1) / 2;
    dmm::FramePtrs off;
    c->L.frame_bytes = frame_layout(cfg, &off);
    char* b = (char*)workspace;
    c->L.base.img_l = (uint8_t*)(b + (size_t)off.img_l);
    c->L.base.img_r = (uint8_t*)(b + (size_t)off.img_r);
    c->L.base.codes_l = (uint32_t*)(b + (size_t)off.codes_l);
    c->L.base.codes_r = (uint32_t*)(b + (size_t)off.codes_r);
    c->L.base.D = (uint8_t*)(b + (size_t)off.D);
    c->L.base.fv = (uint8_t*)(b + (size_t)off.fv);
    c->L.base.fh = (uint8_t*)(b + (size_t)off.fh);
    c->L.base.fwd = (int32_t*)(b + (size_t)off.fwd);
    c->L.base.bwd = (int32_t*)(b + (size_t)off.bwd);
    c->L.base.fwdo = (int32_t*)(b + (size_t)off.fwdo);
    c->L.base.bwdo = (int32_t*)(b + (size_t)off.bwdo);
    c->L.base.labels = (uint8_t*)(b + (size_t)off.labels);
    c->L.base.bounds = (long long*)(b + (size_t)off.bounds);
    c->L.base.energy = (long long*)(b + (size_t)off.energy);
    c->L.base.flag = (int32_t*)(b + (size_t)off.flag);
    c->L.base.rf = (float*)(b + (size_t)off.rf);
    c->L.base.tmap = (uint8_t*)(b + (size_t)off.tmap);
    c->L.base.renergy = (double*)(b + (size_t)off.renergy);
    c->L.base.gfv = (int32_t*)(b + (size_t)off.gfv);
    c->L.base.ggh = (int32_t*)(b + (size_t)off.ggh);
    c->L.base.gom_h = (uint8_t*)(b + (size_t)off.gom_h);
    c->L.base.gom_v = (uint8_t*)(b + (size_t)off.gom_v);
    c->L.W = cfg->width; c->L.H = cfg->height; c->L.K = c->K; c->L.KP = c->KP;
    c->ws = b;
    c->ws_bytes = bytes;
    c->has_cost = new int[cfg->batch]();
    c->iters_done = new int[cfg->batch]();
    c->launches = 0;
    c->profiling = 0;
    c->stop_after_h = 0;
    c->pair_ok = dmm::gen_mode(cfg) ? 0 : pair_range_ok(cfg);
    c->use_pair = 1;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        dmm_destroy(c);
        return DMM_E_CUDA;
    }
    {   // V half-step tensor maps of every frame (tmap.cu)
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        cudaError_t e = cudaSuccess;
        for (int f = 0; f < cfg->batch && e == cudaSuccess; ++f) {
            dmm::FramePtrs P = dmm::frame_ptrs(c->L, f);
            e = dmm::build_vmaps(P.fv, P.D, cfg->width, cfg->height, c->KP, P.tmap);
        }
        if (prev >= 0) cudaSetDevice(prev);
        c->vtma = e == cudaSuccess;   // else the V kernels stage one bulk copy per node
        cudaGetLastError();
    }
    if (dmm::gen_mode(cfg)) {
        // edge-weight table (reading R30), computed on the host in double as
        // the oracle does, uploaded after every frame's vertical weight map
        uint8_t lut[256];
        for (int g = 0; g < 256; ++g) {
            const double v = floor(16.0 * exp(-5.0 * (double)g / 255.0) + 0.5);
            lut[g] = (uint8_t)(v < 1.0 ? 1 : (v > 16.0 ? 16 : v));
        }
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        cudaError_t e = cudaSuccess;
        for (int f = 0; f < cfg->batch && e == cudaSuccess; ++f) {
            dmm::FramePtrs P = dmm::frame_ptrs(c->L, f);
            e = cudaMemcpy(P.gom_v + (size_t)cfg->width * cfg->height, lut, 256, cudaMemcpyHostToDevice);
            if (e == cudaSuccess && !cfg->edge_weights) {   // constant weights: the maps stay 16
                e = cudaMemset(P.gom_h, 16, (size_t)cfg->width * cfg->height);
                if (e == cudaSuccess) e = cudaMemset(P.gom_v, 16, (size_t)cfg->width * cfg->height);
            }
        }
        if (prev >= 0) cudaSetDevice(prev);
        if (e != cudaSuccess) { dmm_destroy(c); return DMM_E_CUDA; }
    }
    *out = c;
    return DMM_OK;
}

void dmm_destroy(dmm_ctx* ctx) {
    if (!ctx) return;
    for (auto& r : ctx->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ctx->pool) cudaEventDestroy(e);
    dmm::shard_release(ctx);
    dmm::refine_release(ctx);
    delete[] ctx->has_cost;
    delete[] ctx->iters_done;
    delete ctx;
}

dmm_status dmm_cost_volume(dmm_ctx* ctx, int frame, const uint8_t* left, const uint8_t* right,
                           int64_t pitch, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st) return st;
    if (!left || !right) { ctx->err = "null image"; return DMM_E_ARG; }
    if (pitch < ctx->cfg.width) { ctx->err = "pitch < width"; return DMM_E_SHAPE; }
    cudaStream_t s = (cudaStream_t)stream;
    if (rowcol(ctx)) {
        Timed t(ctx, 1, s, ctx->sh.world > 1 ? 3 : 2);
        if ((st = dmm::shard_cost_volume(ctx, left, right, pitch, s))) return st;
    } else {
        { Timed t(ctx, 0, s); dmm::launch_census(ctx->L, frame, 1, ctx->cfg.census_radius, pitch, left, right, s); }
        { Timed t(ctx, 1, s); dmm::launch_cost(ctx->L, frame, 1, ctx->cfg.d_min, ctx->oob, s); }
        if (ctx->cfg.edge_weights) dmm::gen_weights(ctx, frame, left, pitch, s);
    }
    if ((st = check_launch(ctx, "cost_volume"))) return st;
    ctx->has_cost[frame] = 1;
    ctx->iters_done[frame] = 0;
    return DMM_OK;
}

dmm_status dmm_refine(dmm_ctx* ctx, int frame, const dmm_refine_params* prm, float* u_out, double* energy,
                      void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st || (st = not_sharded(ctx, "dmm_refine"))) return st;
    if (!prm || prm->warps < 0 || prm->iters < 0 || prm->iters > 4096 || !(prm->h > 0.0) || !(prm->tau > 0.0) ||
        !(prm->sigma > 0.0) || !(prm->eps >= 0.0 && prm->eps <= 1.0) || !(prm->delta >= 0.0) || !(prm->C >= 0.0)) {
        ctx->err = "bad refinement parameters";
        return DMM_E_ARG;
    }
    if (ctx->iters_done[frame] < 1) { ctx->err = "refine before solve (needs the discrete labelling)"; return DMM_E_STATE; }
    cudaStream_t s = (cudaStream_t)stream;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    if (energy && (st = cuda_err(ctx, cudaMemsetAsync(P.renergy, 0, 8, s), "memset"))) return st;
    {
        Timed t(ctx, 5, s, 0);
        if ((st = dmm::refine_run(ctx, frame, prm, u_out, energy ? P.renergy : nullptr, s))) return st;
    }
    if (energy) {
        if ((st = cuda_err(ctx, cudaMemcpyAsync(energy, P.renergy, 8, cudaMemcpyDeviceToHost, s), "d2h"))) return st;
        if ((st = cuda_err(ctx, cudaStreamSynchronize(s), "sync"))) return st;
    }
    return DMM_OK;
}

dmm_status dmm_flow_refine(dmm_ctx* ctx, int frame, int32_t v_min, const dmm_refine_params* prm, float* u1_out,
                           float* u2_out, double* energy, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame, 2);
    if (st || (st = not_sharded(ctx, "dmm_flow_refine"))) return st;
    if (!prm || prm->warps < 0 || prm->iters < 0 || prm->iters > 4096 || !(prm->h > 0.0) || !(prm->tau > 0.0) ||
        !(prm->sigma > 0.0) || !(prm->eps >= 0.0 && prm->eps <= 1.0) || !(prm->delta >= 0.0) || !(prm->C >= 0.0)) {
        ctx->err = "bad refinement parameters";
        return DMM_E_ARG;
    }
    if (ctx->iters_done[frame] < 1 || ctx->iters_done[frame + 1] < 1) {
        ctx->err = "flow refine before both layers are solved";
        return DMM_E_STATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    if (energy && (st = cuda_err(ctx, cudaMemsetAsync(P.renergy, 0, 8, s), "memset"))) return st;
    {
        Timed t(ctx, 5, s, 0);
        if ((st = dmm::refine_flow_run(ctx, frame, (double)ctx->cfg.d_min, (double)v_min, prm, u1_out, u2_out,
                                       energy ? P.renergy : nullptr, s)))
            return st;
    }
    if (energy) {
        if ((st = cuda_err(ctx, cudaMemcpyAsync(energy, P.renergy, 8, cudaMemcpyDeviceToHost, s), "d2h"))) return st;
        if ((st = cuda_err(ctx, cudaStreamSynchronize(s), "sync"))) return st;
    }
    return DMM_OK;
}

dmm_status dmm_flow_cost_volume(dmm_ctx* ctx, int frame, const uint8_t* left, const uint8_t* right, int64_t pitch,
                                int32_t v_min, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame, 2);
    if (st || (st = not_sharded(ctx, "dmm_flow_cost_volume"))) return st;
    if (!left || !right) { ctx->err = "null image"; return DMM_E_ARG; }
    if (pitch < ctx->cfg.width) { ctx->err = "pitch < width"; return DMM_E_SHAPE; }
    if (!dmm::flow_k_ok(ctx->K)) { ctx->err = "flow window: K must be 16, 32, 48 or 64"; return DMM_E_ARG; }
    cudaStream_t s = (cudaStream_t)stream;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    dmm::FramePtrs P2 = dmm::frame_ptrs(ctx->L, frame + 1);
    { Timed t(ctx, 0, s); dmm::launch_census(ctx->L, frame, 1, ctx->cfg.census_radius, pitch, left, right, s); }
    {
        Timed t(ctx, 1, s);
        dmm::launch_flow_costs(P.codes_l, P.codes_r, ctx->cfg.width, ctx->cfg.height, ctx->K, ctx->KP, ctx->cfg.d_min,
                               v_min, ctx->oob, P.D, P2.D, s);
    }
    if ((st = check_launch(ctx, "flow cost volume"))) return st;
    for (int f = frame; f < frame + 2; ++f) { ctx->has_cost[f] = 1; ctx->iters_done[f] = 0; }
    return DMM_OK;
}

dmm_status dmm_solve(dmm_ctx* ctx, int frame, int nframes, int32_t iterations, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame, nframes);
    if (st) return st;
    if (iterations < 1 || iterations > ctx->cfg.max_iters) {
        ctx->err = "iterations must be in [1, max_iters]";
        return DMM_E_ARG;
    }
    for (int f = frame; f < frame + nframes; ++f)
        if (!ctx->has_cost[f]) { ctx->err = "solve before cost volume"; return DMM_E_STATE; }
    cudaStream_t s = (cudaStream_t)stream;
    if (rowcol(ctx)) {
        if (ctx->stop_after_h) { ctx->err = "stop-after-H is not available on a band-sharded context"; return DMM_E_STATE; }
        if ((st = dmm::shard_solve(ctx, iterations, s))) return st;
        ctx->iters_done[0] = iterations;
        return DMM_OK;
    }
    {   // bound history + energy of every frame: one strided memset
        dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
        const size_t row = (size_t)((char*)P.energy - (char*)P.bounds) + 8;
        if ((st = cuda_err(ctx, cudaMemset2DAsync(P.bounds, ctx->L.frame_bytes, 0, row, nframes, s),
                           "memset bounds")))
            return st;
    }
    for (int t = 0; t < iterations; ++t) {
        for (int v = 0; v < 2; ++v) {
            launch_half(ctx, frame, nframes, t, v, iterations, s);
            if (ctx->stop_after_h) break;
        }
        if (ctx->stop_after_h) break;
    }
    if (ctx->stop_after_h) {   // debug: only f_ after H_1 is meaningful (dmm_copy_dual which = 0)
        if ((st = check_launch(ctx, "solve"))) return st;
        for (int f = frame; f < frame + nframes; ++f) ctx->iters_done[f] = kPartial;
        return DMM_OK;
    }
    {
        Timed tm(ctx, 4, s, dmm::gen_mode(&ctx->cfg) ? 0 : 1);
        if (dmm::gen_mode(&ctx->cfg))
            dmm::gen_energy(ctx, frame, nframes, nullptr, nullptr, s);
        else
            dmm::launch_energy(ctx->L, frame, nframes, ctx->cfg.w_h, ctx->cfg.w_v, ctx->cfg.trunc,
                               ctx->cfg.frac_bits, nullptr, nullptr, s);
    }
    if ((st = check_launch(ctx, "solve"))) return st;
    for (int f = frame; f < frame + nframes; ++f) ctx->iters_done[f] = iterations;
    return DMM_OK;
}

dmm_status dmm_result(dmm_ctx* ctx, int frame, int64_t* energy, int64_t* bound,
                      int64_t* bound_history, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st) return st;
    const int it = ctx->iters_done[frame];
    if (it == kPartial) { ctx->err = "partial (debug stop-after-H) solve has no result"; return DMM_E_STATE; }
    if (it < 1) { ctx->err = "result before solve"; return DMM_E_STATE; }
    cudaStream_t s = (cudaStream_t)stream;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    long long* bptr = rowcol(ctx) ? ctx->sh.bounds : P.bounds;
    long long* eptr = rowcol(ctx) ? ctx->sh.bounds + 2 * it : P.energy;
    long long e = 0;
    if (energy &&
        (st = cuda_err(ctx, cudaMemcpyAsync(&e, eptr, 8, cudaMemcpyDeviceToHost, s), "d2h")))
        return st;
    long long hist[2 * 1024];
    if ((st = cuda_err(ctx, cudaMemcpyAsync(hist, bptr, 8 * 2 * (size_t)it, cudaMemcpyDeviceToHost, s),
                       "d2h bounds")))
        return st;
    if ((st = cuda_err(ctx, cudaStreamSynchronize(s), "sync"))) return st;
    if (energy) *energy = e;
    if (bound) *bound = hist[2 * it - 1];
    if (bound_history) memcpy(bound_history, hist, 8 * 2 * (size_t)it);
    return DMM_OK;
}

dmm_status dmm_copy_labels(dmm_ctx* ctx, int frame, uint8_t* labels, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st) return st;
    if (!labels) return DMM_E_ARG;
    if (ctx->iters_done[frame] < 1) { ctx->err = "labels before solve"; return DMM_E_STATE; }
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    return cuda_err(ctx,
                    cudaMemcpyAsync(labels, rowcol(ctx) ? ctx->sh.labels_full : P.labels,
                                    (size_t)ctx->L.W * ctx->L.H,
                                    cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
                    "copy labels");
}

dmm_status dmm_copy_codes(dmm_ctx* ctx, int frame, int which, uint32_t* dst, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st) return st;
    if (!dst || (which != 0 && which != 1)) return DMM_E_ARG;
    if (!ctx->has_cost[frame]) return DMM_E_STATE;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    if (rowcol(ctx)) { P.codes_l = ctx->sh.codes_l; P.codes_r = ctx->sh.codes_r; }
    return cuda_err(ctx,
                    cudaMemcpyAsync(dst, which ? P.codes_r : P.codes_l, 4 * (size_t)ctx->L.W * ctx->L.H,
                                    cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
                    "copy codes");
}

dmm_status dmm_copy_cost_volume(dmm_ctx* ctx, int frame, uint8_t* dst, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st || (st = not_sharded(ctx, "dmm_copy_cost_volume"))) return st;
    if (st) return st;
    if (!dst) return DMM_E_ARG;
    if (!ctx->has_cost[frame]) return DMM_E_STATE;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    dmm::launch_unpad_u8(P.D, dst, (long long)ctx->L.W * ctx->L.H, ctx->K, ctx->KP, (cudaStream_t)stream);
    return check_launch(ctx, "copy cost volume");
}

dmm_status dmm_copy_dual(dmm_ctx* ctx, int frame, int which, int32_t* dst, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st || (st = not_sharded(ctx, "dmm_copy_dual"))) return st;
    if (st) return st;
    if (!dst || (which != 0 && which != 1)) return DMM_E_ARG;
    if (ctx->iters_done[frame] == 0 || (ctx->iters_done[frame] == kPartial && which != 0)) return DMM_E_STATE;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    if (dmm::gen_mode(&ctx->cfg))
        dmm::launch_decode_dense(which ? P.ggh : P.gfv, which ? P.D : nullptr, ctx->cfg.frac_bits, dst,
                                 (long long)ctx->L.W * ctx->L.H, ctx->K, ctx->KP, (cudaStream_t)stream);
    else
        dmm::launch_decode_rec(which ? P.fh : P.fv, which ? P.D : nullptr, ctx->cfg.frac_bits, dst,
                               (long long)ctx->L.W * ctx->L.H, ctx->K, ctx->KP, (cudaStream_t)stream);
    return check_launch(ctx, "copy dual");
}

dmm_status dmm_run_host(dmm_ctx* ctx, int frame, const uint8_t* left_host, const uint8_t* right_host,
                        int32_t iterations, uint8_t* labels_host, int64_t* energy, int64_t* bound,
                        void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st) return st;
    if (!left_host || !right_host || !labels_host) return DMM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    if (rowcol(ctx)) { P.img_l = ctx->sh.img_l; P.img_r = ctx->sh.img_r; P.labels = ctx->sh.labels_full; }
    const size_t px = (size_t)ctx->L.W * ctx->L.H;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(P.img_l, left_host, px, cudaMemcpyHostToDevice, s), "h2d")))
        return st;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(P.img_r, right_host, px, cudaMemcpyHostToDevice, s), "h2d")))
        return st;
    if ((st = dmm_cost_volume(ctx, frame, P.img_l, P.img_r, ctx->L.W, stream))) return st;
    if ((st = dmm_solve(ctx, frame, 1, iterations, stream))) return st;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(labels_host, P.labels, px, cudaMemcpyDeviceToHost, s), "d2h")))
        return st;
    return dmm_result(ctx, frame, energy, bound, nullptr, stream);
}

dmm_status dmm_cost_volume_frames(dmm_ctx* ctx, int frame, int nframes, const uint8_t* left,
                                  const uint8_t* right, int64_t pitch, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame, nframes);
    if (st || (st = not_sharded(ctx, "dmm_cost_volume_frames"))) return st;
    if (st) return st;
    if (!left || !right) { ctx->err = "null image"; return DMM_E_ARG; }
    if (pitch < ctx->cfg.width) { ctx->err = "pitch < width"; return DMM_E_SHAPE; }
    cudaStream_t s = (cudaStream_t)stream;
    { Timed t(ctx, 0, s); dmm::launch_census(ctx->L, frame, nframes, ctx->cfg.census_radius, pitch, left, right, s); }
    { Timed t(ctx, 1, s); dmm::launch_cost(ctx->L, frame, nframes, ctx->cfg.d_min, ctx->oob, s); }
    if (ctx->cfg.edge_weights)
        for (int f = 0; f < nframes; ++f) dmm::gen_weights(ctx, frame + f, left + (size_t)f * pitch * ctx->L.H, pitch, s);
    if ((st = check_launch(ctx, "cost_volume_frames"))) return st;
    for (int f = frame; f < frame + nframes; ++f) { ctx->has_cost[f] = 1; ctx->iters_done[f] = 0; }
    return DMM_OK;
}

dmm_status dmm_run_host_frames(dmm_ctx* ctx, int frame, int nframes, const uint8_t* left_host,
                               const uint8_t* right_host, int32_t iterations, uint8_t* labels_host,
                               int64_t* energy, int64_t* bound, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame, nframes);
    if (st || (st = not_sharded(ctx, "dmm_run_host_frames"))) return st;
    if (st) return st;
    if (!left_host || !right_host || !labels_host || !energy || !bound) return DMM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    const size_t px = (size_t)ctx->L.W * ctx->L.H, fb = ctx->L.frame_bytes;
    // host [nframes][px] <-> the frames' staging / label arrays (stride frame_bytes)
    if ((st = cuda_err(ctx, cudaMemcpy2DAsync(P.img_l, fb, left_host, px, px, nframes, cudaMemcpyHostToDevice, s),
                       "h2d")))
        return st;
    if ((st = cuda_err(ctx, cudaMemcpy2DAsync(P.img_r, fb, right_host, px, px, nframes, cudaMemcpyHostToDevice, s),
                       "h2d")))
        return st;
    { Timed t(ctx, 0, s); dmm::launch_census(ctx->L, frame, nframes, ctx->cfg.census_radius, ctx->L.W, nullptr, nullptr, s); }
    { Timed t(ctx, 1, s); dmm::launch_cost(ctx->L, frame, nframes, ctx->cfg.d_min, ctx->oob, s); }
    if (ctx->cfg.edge_weights)
        for (int f = frame; f < frame + nframes; ++f) dmm::gen_weights(ctx, f, dmm::frame_ptrs(ctx->L, f).img_l, ctx->L.W, s);
    if ((st = check_launch(ctx, "run_host_frames"))) return st;
    for (int f = frame; f < frame + nframes; ++f) { ctx->has_cost[f] = 1; ctx->iters_done[f] = 0; }
    if ((st = dmm_solve(ctx, frame, nframes, iterations, stream))) return st;
    if ((st = cuda_err(ctx, cudaMemcpy2DAsync(labels_host, px, P.labels, fb, px, nframes, cudaMemcpyDeviceToHost, s),
                       "d2h")))
        return st;
    if ((st = cuda_err(ctx, cudaMemcpy2DAsync(energy, 8, P.energy, fb, 8, nframes, cudaMemcpyDeviceToHost, s),
                       "d2h energy")))
        return st;
    if ((st = cuda_err(ctx, cudaMemcpy2DAsync(bound, 8, P.bounds + 2 * iterations - 1, fb, 8, nframes,
                                              cudaMemcpyDeviceToHost, s),
                       "d2h bound")))
        return st;
    return cuda_err(ctx, cudaStreamSynchronize(s), "sync");
}

dmm_status dmm_buffer_ptr(dmm_ctx* ctx, int frame, int which, void** ptr, size_t* bytes, int* bytes_per_pixel) {
    dmm_status st = frame_ok(ctx, frame);
    if (st || (st = not_sharded(ctx, "dmm_buffer_ptr"))) return st;
    if (st) return st;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    const size_t px = (size_t)ctx->L.W * ctx->L.H;
    void* p = nullptr;
    int bpp = 0;
    size_t n = 0;
    switch (which) {
        case DMM_BUF_D: p = P.D; bpp = ctx->KP; n = px * bpp; break;
        case DMM_BUF_FV: p = P.fv; bpp = dmm::rec_bytes(ctx->KP); n = px * bpp; break;
        case DMM_BUF_FH: p = P.fh; bpp = dmm::rec_bytes(ctx->KP); n = px * bpp; break;
        case DMM_BUF_LABELS: p = P.labels; bpp = 1; n = px; break;
        case DMM_BUF_BOUNDS: p = P.bounds; bpp = 0; n = 8 * 2 * (size_t)ctx->cfg.max_iters; break;
        default: ctx->err = "unknown buffer"; return DMM_E_ARG;
    }
    if (ptr) *ptr = p;
    if (bytes) *bytes = n;
    if (bytes_per_pixel) *bytes_per_pixel = bpp;
    return DMM_OK;
}

dmm_status dmm_import_cost_volume(dmm_ctx* ctx, int frame, const uint8_t* D_dense, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st || (st = not_sharded(ctx, "dmm_import_cost_volume"))) return st;
    if (st) return st;
    if (!D_dense) return DMM_E_ARG;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    dmm::launch_pad_u8(D_dense, P.D, (long long)ctx->L.W * ctx->L.H, ctx->K, ctx->KP, (cudaStream_t)stream);
    if ((st = check_launch(ctx, "import cost volume"))) return st;
    ctx->has_cost[frame] = 1;
    ctx->iters_done[frame] = 0;
    return DMM_OK;
}

dmm_status dmm_half_step(dmm_ctx* ctx, int frame, int nframes, int32_t t, int vertical, int32_t iterations,
                         void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame, nframes);
    if (st) return st;
    if (iterations < 1 || iterations > ctx->cfg.max_iters || t < 0 || t >= iterations ||
        (vertical != 0 && vertical != 1)) {
        ctx->err = "bad half-step index";
        return DMM_E_ARG;
    }
    for (int f = frame; f < frame + nframes; ++f)
        if (!ctx->has_cost[f]) { ctx->err = "half step before cost volume"; return DMM_E_STATE; }
    cudaStream_t s = (cudaStream_t)stream;
    if (rowcol(ctx)) {     // this rank's band; the caller moves the records (dmm_shard_plan)
        if (frame != 0 || nframes != 1) return DMM_E_ARG;
        if ((st = cuda_err(ctx, cudaMemsetAsync(ctx->sh.bounds + 2 * t + vertical, 0, 8, s), "memset bound slot")))
            return st;
        if ((st = dmm::shard_half_step(ctx, t, vertical, iterations, s))) return st;
        if (vertical && t == iterations - 1) ctx->iters_done[0] = iterations;
        return DMM_OK;
    }
    {   // reset this half-step's bound slot of every frame
        dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
        if ((st = cuda_err(ctx, cudaMemset2DAsync(P.bounds + 2 * t + vertical, ctx->L.frame_bytes, 0, 8,
                                                  nframes, s),
                           "memset bound slot")))
            return st;
    }
    launch_half(ctx, frame, nframes, t, vertical, iterations, s);
    if ((st = check_launch(ctx, "half step"))) return st;
    if (vertical && t == iterations - 1)
        for (int f = frame; f < frame + nframes; ++f) ctx->iters_done[f] = iterations;
    return DMM_OK;
}

dmm_status dmm_energy(dmm_ctx* ctx, int frame, int64_t* energy, void* stream) {
    return dmm_energy_of(ctx, frame, nullptr, energy, stream);
}

dmm_status dmm_energy_of(dmm_ctx* ctx, int frame, const uint8_t* labels, int64_t* energy, void* stream) {
    if (!ctx) return DMM_E_ARG;
    DMM_DEVICE_GUARD(ctx);
    dmm_status st = frame_ok(ctx, frame);
    if (st || (st = not_sharded(ctx, "dmm_energy_of"))) return st;
    if (st) return st;
    if (!energy) return DMM_E_ARG;
    if (!ctx->has_cost[frame]) { ctx->err = "energy before cost volume"; return DMM_E_STATE; }
    cudaStream_t s = (cudaStream_t)stream;
    dmm::FramePtrs P = dmm::frame_ptrs(ctx->L, frame);
    int* bad = P.flag;     // set by the kernel if a label is >= K
    long long e = 0;
    int badh = 0;
    if ((st = cuda_err(ctx, cudaMemsetAsync(P.energy, 0, 8, s), "memset energy"))) return st;
    if ((st = cuda_err(ctx, cudaMemsetAsync(bad, 0, 4, s), "memset flag"))) return st;
    {
        Timed tm(ctx, 4, s);
        if (dmm::gen_mode(&ctx->cfg)) {
            dmm::gen_energy(ctx, frame, 1, labels, bad, s);
        } else {
            dmm::launch_energy(ctx->L, frame, 1, ctx->cfg.w_h, ctx->cfg.w_v, ctx->cfg.trunc, ctx->cfg.frac_bits,
                               labels, bad, s);
        }
    }
    if ((st = check_launch(ctx, "energy"))) return st;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(&e, P.energy, 8, cudaMemcpyDeviceToHost, s), "d2h"))) return st;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(&badh, bad, 4, cudaMemcpyDeviceToHost, s), "d2h"))) return st;
    if ((st = cuda_err(ctx, cudaStreamSynchronize(s), "sync"))) return st;
    if (badh) { ctx->err = "label index >= K"; return DMM_E_ARG; }
    *energy = e;
    return DMM_OK;
}

int64_t dmm_launch_count(const dmm_ctx* ctx) { return ctx ? ctx->launches : 0; }

dmm_status dmm_set_tuning(dmm_ctx* ctx, int param, int64_t value) {
    if (!ctx) return DMM_E_ARG;
    if (param == DMM_TUNE_DEBUG_STOP_AFTER_H) { ctx->stop_after_h = value != 0; return DMM_OK; }
    if (param == DMM_TUNE_PAIR) { ctx->use_pair = value != 0; return DMM_OK; }
    if (param == DMM_TUNE_QUERY_PAIR) { ctx->err = ctx->use_pair && ctx->pair_ok ? "pair" : "int32"; return DMM_OK; }
    ctx->err = "unknown tuning parameter";
    return DMM_E_ARG;
}

dmm_status dmm_set_profiling(dmm_ctx* ctx, int enable) {
    if (!ctx) return DMM_E_ARG;
    ctx->profiling = enable != 0;
    return DMM_OK;
}

dmm_status dmm_read_profile(dmm_ctx* ctx, double* ms, int64_t* launches) {
    if (!ctx) return DMM_E_ARG;
    for (int c = 0; c < DMM_PROFILE_CLASSES; ++c) {
        if (ms) ms[c] = 0.0;
        if (launches) launches[c] = 0;
    }
    dmm_status st = DMM_OK;
    for (auto& r : ctx->recs) {
        float t = 0.f;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
        if (e != cudaSuccess && st == DMM_OK) st = cuda_err(ctx, e, "read_profile");
        if (ms) ms[r.cls] += t;
        if (launches) launches[r.cls] += 1;
        ctx->pool.push_back(r.a);
        ctx->pool.push_back(r.b);
    }
    ctx->recs.clear();
    return st;
}

const char* dmm_status_str(dmm_status s) {
    switch (s) {
        case DMM_OK: return "ok";
        case DMM_E_ARG: return "invalid argument";
        case DMM_E_SHAPE: return "shape mismatch";
        case DMM_E_STATE: return "invalid state";
        case DMM_E_CUDA: return "CUDA error";
        case DMM_E_RANGE: return "numeric range";
        case DMM_E_NCCL: return "NCCL error";
    }
    return "unknown";
}

const char* dmm_last_error(const dmm_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

}  // extern "C"
