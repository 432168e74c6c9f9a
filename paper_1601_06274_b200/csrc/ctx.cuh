// ctx.cuh -- the context behind the opaque dmm_ctx handle of include/dmm.h
// (host state only; all arrays live in the caller's device workspace).
#pragma once
#include <string>
#include <vector>

#include "../../include/dmm.h"
#include "dmm_internal.cuh"

// Band-sharded context state (dmm_shard): rank r owns row band
// [rb[r], rb[r+1]) for the H half-steps and column band [cb[r], cb[r+1]) for
// the V half-steps; the H band's records are stored in column segments (one
// per destination rank) so that every block of the all-to-all transpose is
// contiguous on both sides.
struct ShardState {
    int mode = -1;          // -1 unsharded, DMM_SHARD_FRAMES, DMM_SHARD_ROWCOL
    int rank = 0, world = 1;
    void* comm = nullptr;   // ncclComm_t (nullptr: external transport, dmm_shard_plan)
    std::vector<int> rb, cb;
    dmm::Layout Lh, Lv;     // the H band (W x hr, segmented records) and the V band (wc x H) as frames
    int* segx = nullptr;    // device copy of cb (PassArgs::segx)
    uint8_t* labels_full = nullptr;   // [H][W]
    uint8_t* lab_gather = nullptr;    // [H][W]: block s = the V band labels [H][wc_s] of rank s
    uint8_t* img_l = nullptr;
    uint8_t* img_r = nullptr;
    uint32_t* codes_l = nullptr;
    uint32_t* codes_r = nullptr;
    long long* bounds = nullptr;      // [2*max_iters] then energy: one all-reduce
    int vtma = 0;                     // V band tensor maps encoded
};

// The captured CUDA graph of one refinement warp (refine.cu), cached per
// (frame, parameters).
struct RefineGraph {
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cap = nullptr;
    int frame = -1;
    int launches_per_warp = 0;
    dmm_refine_params prm{};
    float* rf = nullptr;
};

struct dmm_ctx {
    dmm_config cfg;
    int K, KP, device, oob;
    dmm::Layout L;
    char* ws;
    size_t ws_bytes;
    // per-frame host state
    int* has_cost;
    int* iters_done;
    long long launches;
    std::string err;
    // event profiling (dmm_set_profiling)
    int profiling;
    int stop_after_h;     // debug: dmm_solve runs only the first H half-step
    int pair_ok;          // configuration passes pair_range_ok
    int use_pair;         // DMM_TUNE_PAIR (default 1): packed chain-pair kernels when pair_ok
    int vtma = 0;         // the frames' V tensor maps are encoded (tmap.cu)
    struct Rec { int cls; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    ShardState sh;
    RefineGraph rg;       // stereo refinement
    RefineGraph rgf;      // flow refinement
};

namespace dmm {
// capi.cu: one half-step of iteration t on `nframes` frames of layout L
// (records in nseg column segments when nseg > 1); returns a launch error.
dmm_status launch_half_on(dmm_ctx* ctx, const Layout& L, int frame, int nframes, int t, int v, int iterations,
                          int nseg, const int* segx, cudaStream_t s);
dmm_status cuda_status(dmm_ctx* ctx, cudaError_t e, const char* where);
// shard.cu
dmm_status shard_cost_volume(dmm_ctx* ctx, const uint8_t* left, const uint8_t* right, int64_t pitch,
                             cudaStream_t s);
dmm_status shard_solve(dmm_ctx* ctx, int iterations, cudaStream_t s);
dmm_status shard_half_step(dmm_ctx* ctx, int t, int vertical, int iterations, cudaStream_t s);
void shard_release(dmm_ctx* ctx);
// hmg.cu (general pairwise model, NEXT-3)
bool gen_mode(const dmm_config* c);
int genR_host(const dmm_config& c, int d);
void gen_weights(dmm_ctx* ctx, int frame, const uint8_t* left, int64_t pitch, cudaStream_t s);
void gen_half(dmm_ctx* ctx, int frame, int nframes, int t, int v, int iterations, cudaStream_t s);
void gen_energy(dmm_ctx* ctx, int frame, int nframes, const uint8_t* labels, int32_t* bad, cudaStream_t s);
// refine.cu
size_t refine_bytes(int W, int H);
dmm_status refine_run(dmm_ctx* ctx, int frame, const dmm_refine_params* prm, float* out, double* energy_dev,
                      cudaStream_t s);
void refine_release(dmm_ctx* ctx);
dmm_status refine_flow_run(dmm_ctx* ctx, int frame, double u1_min, double u2_min, const dmm_refine_params* prm,
                           float* out1, float* out2, double* energy_dev, cudaStream_t s);
}  // namespace dmm
