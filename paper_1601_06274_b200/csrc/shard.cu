// shard.cu -- multi-GPU sharding behind the C ABI:
// dmm_nccl_unique_id / dmm_shard and the band-sharded solve of one frame.
//
// ROWCOL mode: rank r owns the row band [rb[r], rb[r+1]) for the H half-steps
// and the column band [cb[r], cb[r+1]) for the V half-steps.  Chains of one
// orientation are independent ("decoupled for all horizontal (resp. vertical)
// chains"), so each half-step is local; between half-steps the records
// are transposed with one all-to-all of grouped ncclSend / ncclRecv owned by
// the library:
//   after H: f_ (the V unaries) row band -> column band,
//   after V: D*2^F + g_ (the H unaries) column band -> row band.
// The H band's records are stored in column segments (segment s = the block
// for rank s, [hr][wc_s] row-major; PassArgs::segx), so the leaf kernels'
// bulk stores write each destination's block contiguously -- the send buffer
// IS the output, and the receive lands directly in the V band's row range:
// no pack / unpack copies.  Bounds (sums of chain optima) and the
// energy are int64 partial sums combined by one ncclAllReduce; the labels
// (written by the last V in column bands) are all-gathered.  NCCL is loaded
// with dlopen when a communicator is first created, so the library itself
// has no link-time NCCL dependency (CPU-only hosts load it for the host-only
// entry points).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "ctx.cuh"

namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
    bool tried = false, ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.tried) return api;
    api.tried = true;
    // the process's NCCL if one is loaded (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
#define DMM_SYM(name, field) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    DMM_SYM("ncclGetUniqueId", GetUniqueId);
    DMM_SYM("ncclCommInitRank", CommInitRank);
    DMM_SYM("ncclCommDestroy", CommDestroy);
    DMM_SYM("ncclSend", Send);
    DMM_SYM("ncclRecv", Recv);
    DMM_SYM("ncclGroupStart", GroupStart);
    DMM_SYM("ncclGroupEnd", GroupEnd);
    DMM_SYM("ncclAllReduce", AllReduce);
    DMM_SYM("ncclGetErrorString", GetErrorString);
#undef DMM_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
             api.GroupEnd && api.AllReduce && api.GetErrorString;
    return api;
}

dmm_status nccl_err(dmm_ctx* ctx, ncclResult_t r, const char* where) {
    if (r == ncclSuccess) return DMM_OK;
    if (ctx) ctx->err = std::string(where) + ": " + nccl().GetErrorString(r);
    return DMM_E_NCCL;
}

// ----------------------------------------------------------- band layout
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int kp_of(int K) {
    int lpl = 1;
    while (32 * lpl < K) lpl *= 2;
    return 32 * lpl;
}

// [start, stop) of band k of n items over world ranks (sizes differ by <= 1;
// the first n % world bands are one longer) -- sharding.bands in Python.
int band_start(int n, int world, int k) {
    const int q = n / world, r = n % world;
    return k * q + (k < r ? k : r);
}

struct ShardOff {
    size_t img_l, img_r, codes_l, codes_r;
    size_t Dh, fhh, fvh, Dv, fvv, fhv;
    size_t fwd, bwd, fwdo, bwdo;
    size_t labels_v, labels_full, lab_gather, bounds, flag, segx, tmap;
    size_t total;
    int r0, r1, c0, c1;
};

// Byte offsets (from the workspace base) of a ROWCOL rank's arrays.  With
// world == 1 the V band is the H band (same frame, no exchange): aliased.
ShardOff shard_offsets(const dmm_config* c, int rank, int world) {
    ShardOff o{};
    const size_t W = c->width, H = c->height, KP = kp_of(c->d_max - c->d_min + 1);
    const size_t REC = dmm::rec_bytes((int)KP);
    o.r0 = band_start((int)H, world, rank);
    o.r1 = band_start((int)H, world, rank + 1);
    o.c0 = band_start((int)W, world, rank);
    o.c1 = band_start((int)W, world, rank + 1);
    const size_t hr = o.r1 - o.r0, wc = o.c1 - o.c0;
    const size_t pxh = hr * W, pxv = H * wc, pxmax = pxh > pxv ? pxh : pxv;
    size_t p = 0;
    auto take = [&](size_t bytes) { size_t r = p; p = align256(p + bytes); return r; };
    o.img_l = take(W * H);
    o.img_r = take(W * H);
    o.codes_l = take(4 * W * H);
    o.codes_r = take(4 * W * H);
    o.Dh = take(pxh * KP);
    o.fhh = take(pxh * REC);
    o.fvh = take(pxh * REC);
    if (world > 1) {
        o.Dv = take(pxv * KP);
        o.fvv = take(pxv * REC);
        o.fhv = take(pxv * REC);
    } else {
        o.Dv = o.Dh; o.fvv = o.fvh; o.fhv = o.fhh;
    }
    o.fwd = take(4 * pxmax * KP);
    o.bwd = take(4 * pxmax * KP);
    o.fwdo = take(8 * pxmax);
    o.bwdo = take(8 * pxmax);
    o.labels_v = take(pxv);
    o.labels_full = take(W * H);
    o.lab_gather = take(W * H);
    o.bounds = take(8 * (2 * (size_t)c->max_iters + 1));   // bound history, then the energy
    o.flag = take(8);
    o.segx = take(4 * ((size_t)world + 1));
    o.tmap = take(dmm::kTmapBytes);
    o.total = p;
    return o;
}

bool rowcol_ok(const dmm_config* c, int world) {
    return world >= 1 && world <= 64 && c->batch == 1 && c->width / world >= 16 && c->height / world >= 1;
}

// One all-to-all phase: 0 = after H (f_ records, H band segment s -> rank s's
// V band rows [r0, r1)), 1 = after V (D*2^F + g_ records back).
int plan(const dmm_config* c, int rank, int world, int phase, dmm_xfer* out, int max) {
    const ShardOff me = shard_offsets(c, rank, world);
    const size_t REC = dmm::rec_bytes(kp_of(c->d_max - c->d_min + 1));
    const size_t hr = me.r1 - me.r0, wc = me.c1 - me.c0;
    int n = 0;
    for (int s = 0; s < world; ++s) {
        const int sc0 = band_start(c->width, world, s), sc1 = band_start(c->width, world, s + 1);
        const int sr0 = band_start(c->height, world, s), sr1 = band_start(c->height, world, s + 1);
        dmm_xfer x;
        x.peer = s;
        if (phase == 0) {
            // send: my H band's segment s ([hr][wc_s], segment base = sc0 * hr records)
            x.send_offset = (int64_t)(me.fvh + (size_t)sc0 * hr * REC);
            x.send_bytes = (int64_t)(hr * (size_t)(sc1 - sc0) * REC);
            // recv: rank s's rows [sr0, sr1) of my V band ([H][wc] row-major)
            x.recv_offset = (int64_t)(me.fvv + (size_t)sr0 * wc * REC);
            x.recv_bytes = (int64_t)((size_t)(sr1 - sr0) * wc * REC);
        } else {
            x.send_offset = (int64_t)(me.fhv + (size_t)sr0 * wc * REC);
            x.send_bytes = (int64_t)((size_t)(sr1 - sr0) * wc * REC);
            x.recv_offset = (int64_t)(me.fhh + (size_t)sc0 * hr * REC);
            x.recv_bytes = (int64_t)(hr * (size_t)(sc1 - sc0) * REC);
        }
        if (n < max && out) out[n] = x;
        ++n;
    }
    return n;
}

// ------------------------------------------------------------- kernels
// Assemble the full-frame labelling from the all-gathered V band blocks
// (block s = [H][wc_s] at byte H * cb[s]).
__global__ void assemble_labels_kernel(const uint8_t* __restrict__ gath, uint8_t* __restrict__ full, const int* cb,
                                       int world, int W, int H) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < W * H; q += gridDim.x * blockDim.x) {
        const int y = q / W, x = q - y * W;
        int s = 0;
        while (x >= cb[s + 1]) ++s;
        const int wc = cb[s + 1] - cb[s];
        full[q] = gath[(size_t)H * cb[s] + (size_t)y * wc + (x - cb[s])];
    }
}

// Energy (Eq.3, scaled by 2^F) of the rows [r0, r0 + hr) of a full-frame
// labelling against the H band's cost volume: unaries and horizontal edges of
// these rows, vertical edges (y, y+1) for y in the band (each edge once).
__global__ void __launch_bounds__(256)
energy_band_kernel(const uint8_t* __restrict__ Dh, const uint8_t* __restrict__ lab, int W, int H, int K, int KP,
                   int r0, int hr, int w_h, int w_v, int T, int fbits, long long* energy) {
    long long e = 0;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < W * hr; q += gridDim.x * blockDim.x) {
        const int yl = q / W, x = q - yl * W, y = r0 + yl;
        const int l = lab[(size_t)y * W + x];
        e += Dh[(size_t)q * KP + min(l, K - 1)];
        if (x + 1 < W) e += (long long)w_h * min(abs(l - (int)lab[(size_t)y * W + x + 1]), T);
        if (y + 1 < H) e += (long long)w_v * min(abs(l - (int)lab[(size_t)(y + 1) * W + x]), T);
    }
    for (int d = 16; d > 0; d >>= 1) e += __shfl_down_sync(0xffffffffu, e, d);
    __shared__ long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        atomicAdd(reinterpret_cast<unsigned long long*>(energy), (unsigned long long)(t << fbits));
    }
}

dmm_status exchange(dmm_ctx* ctx, int phase, cudaStream_t s) {
    ShardState& sh = ctx->sh;
    if (sh.world == 1) return DMM_OK;    // aliased: the V band is the H band
    std::vector<dmm_xfer> xs(sh.world);
    plan(&ctx->cfg, sh.rank, sh.world, phase, xs.data(), sh.world);
    dmm_status st;
    // own block: a device copy
    const dmm_xfer& me = xs[sh.rank];
    if ((st = dmm::cuda_status(ctx, cudaMemcpyAsync(ctx->ws + me.recv_offset, ctx->ws + me.send_offset,
                                                    (size_t)me.send_bytes, cudaMemcpyDeviceToDevice, s),
                               "exchange self copy")))
        return st;
    NcclApi& api = nccl();
    ncclComm_t comm = (ncclComm_t)sh.comm;
    if ((st = nccl_err(ctx, api.GroupStart(), "ncclGroupStart"))) return st;
    for (int p = 0; p < sh.world; ++p) {
        if (p == sh.rank) continue;
        const dmm_xfer& x = xs[p];
        if (x.send_bytes > 0 &&
            (st = nccl_err(ctx, api.Send(ctx->ws + x.send_offset, (size_t)x.send_bytes, ncclUint8, p, comm, s),
                           "ncclSend")))
            return st;
        if (x.recv_bytes > 0 &&
            (st = nccl_err(ctx, api.Recv(ctx->ws + x.recv_offset, (size_t)x.recv_bytes, ncclUint8, p, comm, s),
                           "ncclRecv")))
            return st;
    }
    return nccl_err(ctx, api.GroupEnd(), "ncclGroupEnd");
}

}  // namespace

namespace dmm {

void shard_release(dmm_ctx* ctx) {
    if (ctx->sh.comm) nccl().CommDestroy((ncclComm_t)ctx->sh.comm);
    ctx->sh.comm = nullptr;
}

dmm_status shard_cost_volume(dmm_ctx* ctx, const uint8_t* left, const uint8_t* right, int64_t pitch,
                             cudaStream_t s) {
    ShardState& sh = ctx->sh;
    const dmm_config& c = ctx->cfg;
    // census of the whole frame (cheap: 2 x 4 B per pixel), then the cost
    // volume of this rank's row band and column band only
    Layout Lf = ctx->L;
    Lf.base.img_l = sh.img_l; Lf.base.img_r = sh.img_r;
    Lf.base.codes_l = sh.codes_l; Lf.base.codes_r = sh.codes_r;
    Lf.W = c.width; Lf.H = c.height;
    launch_census(Lf, 0, 1, c.census_radius, pitch, left, right, s);
    const int r0 = sh.rb[sh.rank], hr = sh.rb[sh.rank + 1] - r0;
    const int c0 = sh.cb[sh.rank], wc = sh.cb[sh.rank + 1] - c0;
    launch_cost_rect(sh.codes_l, sh.codes_r, 0, c.width, ctx->K, ctx->KP, c.d_min, ctx->oob, 0, r0, c.width, hr,
                     sh.Lh.base.D, 0, 1, s);
    if (sh.world > 1)
        launch_cost_rect(sh.codes_l, sh.codes_r, 0, c.width, ctx->K, ctx->KP, c.d_min, ctx->oob, c0, 0, wc, c.height,
                         sh.Lv.base.D, 0, 1, s);
    return cuda_status(ctx, cudaGetLastError(), "shard cost volume");
}

dmm_status shard_half_step(dmm_ctx* ctx, int t, int v, int iterations, cudaStream_t s) {
    ShardState& sh = ctx->sh;
    return v ? launch_half_on(ctx, sh.Lv, 0, 1, t, 1, iterations, 1, nullptr, s)
             : launch_half_on(ctx, sh.Lh, 0, 1, t, 0, iterations, sh.world, sh.segx, s);
}

dmm_status shard_solve(dmm_ctx* ctx, int iterations, cudaStream_t s) {
    ShardState& sh = ctx->sh;
    const dmm_config& c = ctx->cfg;
    if (!sh.comm && sh.world > 1) {
        ctx->err = "sharded context without a communicator: drive dmm_half_step + dmm_shard_plan";
        return DMM_E_STATE;
    }
    dmm_status st;
    const size_t nred = 2 * (size_t)iterations + 1;
    if ((st = cuda_status(ctx, cudaMemsetAsync(sh.bounds, 0, 8 * (2 * (size_t)c.max_iters + 1), s), "memset")))
        return st;
    for (int t = 0; t < iterations; ++t) {
        if ((st = shard_half_step(ctx, t, 0, iterations, s))) return st;
        if ((st = exchange(ctx, 0, s))) return st;
        if ((st = shard_half_step(ctx, t, 1, iterations, s))) return st;
        if (t + 1 < iterations && (st = exchange(ctx, 1, s))) return st;
    }
    // labels: the V band blocks of all ranks -> the full frame on every rank
    const size_t H = c.height;
    const int wc = sh.cb[sh.rank + 1] - sh.cb[sh.rank];
    if (sh.world > 1) {
        NcclApi& api = nccl();
        ncclComm_t comm = (ncclComm_t)sh.comm;
        if ((st = cuda_status(ctx, cudaMemcpyAsync(sh.lab_gather + H * sh.cb[sh.rank], sh.Lv.base.labels,
                                                   H * wc, cudaMemcpyDeviceToDevice, s), "labels self copy")))
            return st;
        if ((st = nccl_err(ctx, api.GroupStart(), "ncclGroupStart"))) return st;
        for (int p = 0; p < sh.world; ++p) {
            if (p == sh.rank) continue;
            const size_t wp = sh.cb[p + 1] - sh.cb[p];
            if ((st = nccl_err(ctx, api.Send(sh.Lv.base.labels, H * wc, ncclUint8, p, comm, s), "ncclSend")))
                return st;
            if ((st = nccl_err(ctx, api.Recv(sh.lab_gather + H * sh.cb[p], H * wp, ncclUint8, p, comm, s),
                               "ncclRecv")))
                return st;
        }
        if ((st = nccl_err(ctx, api.GroupEnd(), "ncclGroupEnd"))) return st;
        assemble_labels_kernel<<<4 * 148, 256, 0, s>>>(sh.lab_gather, sh.labels_full, sh.segx, sh.world, c.width,
                                                       c.height);
    } else {
        if ((st = cuda_status(ctx, cudaMemcpyAsync(sh.labels_full, sh.Lv.base.labels, H * c.width,
                                                   cudaMemcpyDeviceToDevice, s), "labels copy")))
            return st;
    }
    // energy of the full labelling over this rank's rows, then one int64
    // all-reduce of [bound history, energy]
    long long* energy = sh.bounds + 2 * iterations;
    const int r0 = sh.rb[sh.rank], hr = sh.rb[sh.rank + 1] - r0;
    int blocks = (c.width * hr + 255) / 256;
    if (blocks > 4 * 148) blocks = 4 * 148;
    if (blocks > 0)
        energy_band_kernel<<<blocks, 256, 0, s>>>(sh.Lh.base.D, sh.labels_full, c.width, c.height, ctx->K, ctx->KP,
                                                  r0, hr, c.w_h, c.w_v, c.trunc, c.frac_bits, energy);
    ctx->launches += sh.world > 1 ? 2 : 1;
    if ((st = cuda_status(ctx, cudaGetLastError(), "shard solve"))) return st;
    if (sh.comm)
        return nccl_err(ctx, nccl().AllReduce(sh.bounds, sh.bounds, nred, ncclInt64, ncclSum, (ncclComm_t)sh.comm, s),
                        "ncclAllReduce");
    return DMM_OK;
}

}  // namespace dmm

extern "C" {

dmm_status dmm_nccl_unique_id(uint8_t out[128]) {
    if (!out) return DMM_E_ARG;
    NcclApi& api = nccl();
    if (!api.ok) return DMM_E_NCCL;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return DMM_E_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out, &id, 128);
    return DMM_OK;
}

size_t dmm_shard_workspace_bytes(const dmm_config* cfg, int rank, int world, int mode) {
    if (!cfg || world < 1 || rank < 0 || rank >= world) return 0;
    if (mode == DMM_SHARD_FRAMES) return dmm_workspace_bytes(cfg);
    if (mode != DMM_SHARD_ROWCOL || !rowcol_ok(cfg, world) || dmm_workspace_bytes(cfg) == 0) return 0;
    return shard_offsets(cfg, rank, world).total;
}

int dmm_shard_plan(const dmm_config* cfg, int rank, int world, int phase, dmm_xfer* out, int max) {
    if (!cfg || world < 1 || rank < 0 || rank >= world || (phase != 0 && phase != 1) || !rowcol_ok(cfg, world))
        return -1;
    return plan(cfg, rank, world, phase, out, max);
}

int64_t dmm_shard_locate(const dmm_config* cfg, int rank, int world, int which, int y, int x) {
    if (!cfg || world < 1 || rank < 0 || rank >= world || !rowcol_ok(cfg, world)) return -1;
    if (y < 0 || y >= cfg->height || x < 0 || x >= cfg->width) return -1;
    const ShardOff o = shard_offsets(cfg, rank, world);
    const size_t REC = dmm::rec_bytes(kp_of(cfg->d_max - cfg->d_min + 1));
    const size_t hr = o.r1 - o.r0, wc = o.c1 - o.c0;
    switch (which) {
        case DMM_LOC_FV_H:
        case DMM_LOC_FH_H: {
            if (y < o.r0 || y >= o.r1) return -1;
            int s = 0;
            while (x >= band_start(cfg->width, world, s + 1)) ++s;
            const int x0 = band_start(cfg->width, world, s), w = band_start(cfg->width, world, s + 1) - x0;
            const size_t q = (size_t)x0 * hr + (size_t)(y - o.r0) * w + (x - x0);
            return (int64_t)((which == DMM_LOC_FV_H ? o.fvh : o.fhh) + q * REC);
        }
        case DMM_LOC_FV_V:
        case DMM_LOC_FH_V: {
            if (x < o.c0 || x >= o.c1) return -1;
            const size_t q = (size_t)y * wc + (x - o.c0);
            return (int64_t)((which == DMM_LOC_FV_V ? o.fvv : o.fhv) + q * REC);
        }
        case DMM_LOC_LABEL_V:
            if (x < o.c0 || x >= o.c1) return -1;
            return (int64_t)(o.labels_v + (size_t)y * wc + (x - o.c0));
        case DMM_LOC_BOUNDS:
            return (int64_t)o.bounds;
    }
    return -1;
}

dmm_status dmm_shard(dmm_ctx* ctx, const uint8_t* id, int rank, int world, int mode) {
    if (!ctx) return DMM_E_ARG;
    if (world < 1 || rank < 0 || rank >= world || (mode != DMM_SHARD_FRAMES && mode != DMM_SHARD_ROWCOL)) {
        ctx->err = "bad rank / world / mode";
        return DMM_E_ARG;
    }
    if (ctx->sh.mode >= 0) { ctx->err = "context already sharded"; return DMM_E_STATE; }
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    struct Restore { int p, d; ~Restore() { if (p != d && p >= 0) cudaSetDevice(p); } } restore{prev, ctx->device};
    ShardState& sh = ctx->sh;
    const dmm_config& c = ctx->cfg;
    if (mode == DMM_SHARD_ROWCOL) {
        if (!rowcol_ok(&c, world)) {
            ctx->err = "ROWCOL needs batch == 1 and bands of >= 16 columns and >= 1 row";
            return DMM_E_ARG;
        }
        if (dmm::gen_mode(&c)) {
            ctx->err = "ROWCOL is not available for the general pairwise model";
            return DMM_E_ARG;
        }
        if (!ctx->pair_ok || !ctx->use_pair) {
            ctx->err = "ROWCOL runs the packed chain-pair kernels: configuration outside their range";
            return DMM_E_ARG;
        }
        const ShardOff o = shard_offsets(&c, rank, world);
        if (o.total > ctx->ws_bytes) { ctx->err = "workspace smaller than dmm_shard_workspace_bytes"; return DMM_E_ARG; }
        char* b = ctx->ws;
        sh.rb.resize(world + 1);
        sh.cb.resize(world + 1);
        for (int k = 0; k <= world; ++k) {
            sh.rb[k] = band_start(c.height, world, k);
            sh.cb[k] = band_start(c.width, world, k);
        }
        sh.img_l = (uint8_t*)(b + o.img_l); sh.img_r = (uint8_t*)(b + o.img_r);
        sh.codes_l = (uint32_t*)(b + o.codes_l); sh.codes_r = (uint32_t*)(b + o.codes_r);
        sh.labels_full = (uint8_t*)(b + o.labels_full);
        sh.lab_gather = (uint8_t*)(b + o.lab_gather);
        sh.bounds = (long long*)(b + o.bounds);
        sh.segx = (int*)(b + o.segx);
        dmm::FramePtrs common{};
        common.img_l = sh.img_l; common.img_r = sh.img_r; common.codes_l = sh.codes_l; common.codes_r = sh.codes_r;
        common.fwd = (int32_t*)(b + o.fwd); common.bwd = (int32_t*)(b + o.bwd);
        common.fwdo = (int32_t*)(b + o.fwdo); common.bwdo = (int32_t*)(b + o.bwdo);
        common.labels = (uint8_t*)(b + o.labels_v);
        common.bounds = sh.bounds;
        common.energy = sh.bounds + 2 * c.max_iters;
        common.flag = (int32_t*)(b + o.flag);
        sh.Lh.base = common;
        sh.Lh.base.D = (uint8_t*)(b + o.Dh); sh.Lh.base.fh = (uint8_t*)(b + o.fhh); sh.Lh.base.fv = (uint8_t*)(b + o.fvh);
        sh.Lh.frame_bytes = 0;
        sh.Lh.W = c.width; sh.Lh.H = o.r1 - o.r0; sh.Lh.K = ctx->K; sh.Lh.KP = ctx->KP;
        sh.Lv.base = common;
        sh.Lv.base.D = (uint8_t*)(b + o.Dv); sh.Lv.base.fv = (uint8_t*)(b + o.fvv); sh.Lv.base.fh = (uint8_t*)(b + o.fhv);
        sh.Lv.frame_bytes = 0;
        sh.Lv.W = o.c1 - o.c0; sh.Lv.H = c.height; sh.Lv.K = ctx->K; sh.Lv.KP = ctx->KP;
        sh.Lv.base.tmap = (uint8_t*)(b + o.tmap);
        sh.Lh.base.tmap = nullptr;
        sh.vtma = dmm::build_vmaps(sh.Lv.base.fv, sh.Lv.base.D, sh.Lv.W, sh.Lv.H, ctx->KP, sh.Lv.base.tmap) ==
                  cudaSuccess;
        cudaGetLastError();
        if (cudaMemcpy(sh.segx, sh.cb.data(), 4 * (world + 1), cudaMemcpyHostToDevice) != cudaSuccess) {
            ctx->err = "segment table upload failed";
            return DMM_E_CUDA;
        }
    }
    if (id) {
        NcclApi& api = nccl();
        if (!api.ok) { ctx->err = "libnccl.so.2 not loadable"; return DMM_E_NCCL; }
        ncclUniqueId uid;
        memcpy(&uid, id, sizeof(uid));
        ncclComm_t comm = nullptr;
        dmm_status st = nccl_err(ctx, api.CommInitRank(&comm, world, uid, rank), "ncclCommInitRank");
        if (st) return st;
        sh.comm = comm;
    }
    sh.mode = mode;
    sh.rank = rank;
    sh.world = world;
    return DMM_OK;
}

}  // extern "C"
