// dmm_internal.cuh -- device-side layout and parameter blocks shared by the
// sm_100a kernels of the hot path (census / cost / chain DP / energy).
//
// HBM layout of one frame:
//   codes  u32 [H][W]           census codes, left and right
//   D      u8  [H][W][KP]       cost volume, label-contiguous, KP = 32*LPL >= K
//   fv     rec [H][W]           f_ = minorant of the H pass (the V pass's unaries)
//   fh     rec [H][W]           D*2^F + g_ (the H pass's unaries), g_ = minorant of the V pass
//   fwd    i32 [H][W][KP]       message scratch: message into a node from the left / top
//   bwd    i32 [H][W][KP]       message scratch: message into a node from the right / bottom
//   fwdo, bwdo i32 [H][W][2]    pair path: per-chain offsets of the packed scratch messages
//   labels u8  [H][W]
// rec = compact lossless K-vector record of REC = 2*KP + 16 bytes:
//   u16 v[KP] | int32 base | 12 B pad,  value(k) = base + v[k], base <= min_k
//   (the int32 kernels store base = min_k, the pair kernels the running offset).
// Lossless because every stored vector has a span (max - min over labels)
// below 2^16 (checked at dmm_create).
// Both chain orientations read a node's K-vector as one contiguous record,
// so H chains (stride REC) and V chains (stride W*REC) are both coalesced.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dmm {

// Labels k >= K (padding up to KP) enter every message as +BIG, so they never
// win a minimum; BIG + any reachable message value stays far below 2^31.
constexpr int kBig = 1 << 29;
constexpr unsigned kFull = 0xffffffffu;

struct FramePtrs {
    uint8_t* img_l;
    uint8_t* img_r;
    uint32_t* codes_l;
    uint32_t* codes_r;
    uint8_t* D;
    uint8_t* fv;
    uint8_t* fh;
    int32_t* fwd;
    int32_t* bwd;
    int32_t* fwdo;       // pair path: the two chain offsets of a packed fwd / bwd message [H][W][2]
    int32_t* bwdo;
    uint8_t* labels;
    long long* bounds;   // [2 * max_iters]
    long long* energy;   // [1]
    int32_t* flag;       // [1] scratch: label-range flag of dmm_energy_of
    float* rf;           // continuous refinement state (refine.cu)
    double* renergy;     // [1] energy of the refined labelling
    // general pairwise model (hmg.cu; only allocated when the config asks for it)
    int32_t* gfv;        // f_            int32 [H][W][KP]
    int32_t* ggh;        // D*2^F + g_    int32 [H][W][KP]
    uint8_t* gom_h;      // edge weights of horizontal edges [H][W]
    uint8_t* gom_v;      // edge weights of vertical edges [H][W], then the 256-entry weight table
    // 2-D TMA tensor maps (CUtensorMap, 128 B each) of the V half-step's
    // record / cost arrays (tmap.cu): [0] fv, 16-row boxes (root ring), [1] fv,
    // 8-row boxes (level ring), [2] fv, kLeafMax-row boxes (leaf), [3] D, kLeafMax-row boxes
    uint8_t* tmap;
};

// Per-frame pointers are base + frame * stride (bytes).
struct Layout {
    FramePtrs base;
    size_t frame_bytes;
    int W, H, K, KP;
};

__host__ __device__ constexpr int rec_bytes(int KP) { return 2 * KP + 16; }

__host__ __device__ inline FramePtrs frame_ptrs(const Layout& L, int f) {
    FramePtrs p = L.base;
    const size_t o = (size_t)f * L.frame_bytes;
    p.img_l += o; p.img_r += o;
    p.codes_l = (uint32_t*)((char*)p.codes_l + o);
    p.codes_r = (uint32_t*)((char*)p.codes_r + o);
    p.D += o;
    p.fv += o;
    p.fh += o;
    p.fwd = (int32_t*)((char*)p.fwd + o);
    p.bwd = (int32_t*)((char*)p.bwd + o);
    p.fwdo = (int32_t*)((char*)p.fwdo + o);
    p.bwdo = (int32_t*)((char*)p.bwdo + o);
    p.labels += o;
    p.bounds = (long long*)((char*)p.bounds + o);
    p.energy = (long long*)((char*)p.energy + o);
    p.flag = (int32_t*)((char*)p.flag + o);
    p.rf = (float*)((char*)p.rf + o);
    p.renergy = (double*)((char*)p.renergy + o);
    p.gfv = (int32_t*)((char*)p.gfv + o);
    p.ggh = (int32_t*)((char*)p.ggh + o);
    p.gom_h += o;
    p.gom_v += o;
    p.tmap += o;
    return p;
}

struct PassArgs {
    Layout L;
    int frame0;
    int fbits;        // F
    int ws;           // w * 2^F
    int wsT;          // w * 2^F * T
    int T;            // effective truncation min(T, K)
    int first;        // H pass of iteration 0: g_ == 0, not read
    int last;         // V pass of the last iteration: write labels
    int bound_slot;   // index into bounds[]
    // H records in column segments (band-sharded contexts, dmm_shard): the
    // records of row c, position p live at segx[s]*H + c*(segx[s+1]-segx[s]) +
    // (p - segx[s]) for the segment s containing p; nseg <= 1: row-major.
    int nseg;
    const int* segx;  // device [nseg + 1]
    int vtma;         // V passes stage chunks with the frame's 2-D tensor maps (FramePtrs::tmap)
};

// kernels (launchers in the .cu files)
void launch_census(const Layout& L, int frame0, int nframes, int radius, int64_t pitch,
                   const uint8_t* left, const uint8_t* right, cudaStream_t s);
void launch_cost(const Layout& L, int frame0, int nframes, int d_min, int oob, cudaStream_t s);
// Cost volume of the rectangle [x0, x0+w) x [y0, y0+h) of nframes frames:
// codes are full-frame rows of W (frame stride code_fstride elements), D rows
// of the rectangle have pitch w*KP (frame stride d_fstride bytes).
void launch_cost_rect(const uint32_t* codes_l, const uint32_t* codes_r, size_t code_fstride, int W, int K, int KP,
                      int d_min, int oob, int x0, int y0, int w, int h, uint8_t* D, size_t d_fstride, int nframes,
                      cudaStream_t s);
// One H (vertical = 0) or V (vertical = 1) half-step over all chains, launched
// in waves of `wave` chains (0 = all at once); returns nothing, launches
// hm_launches_per_pass() kernels.
void launch_hm_pass(const PassArgs& a, int vertical, int nframes, int wave, cudaStream_t s);
int hm_launches_per_pass(const PassArgs& a, int vertical, int wave);
// The same half-step on chain pairs in packed 16-bit arithmetic (hm2.cu);
// valid when the configuration passes the pair range check (capi.cu).
void launch_hm2_pass(const PassArgs& a, int vertical, int nframes, cudaStream_t s);
int hm2_launches_per_pass(const PassArgs& a, int vertical);
// labels == nullptr: the frames' own labels; else a caller labelling u8 [H][W]
// (one frame); bad (nullable) is set to 1 if a label is >= K.
// Optimistic decoupled flow costs (flow.cu): f1 -> D1 [H][W][KP], f2 -> D2;
// K in {16, 32, 48, 64} (flow_k_ok).
bool flow_k_ok(int K);
void launch_flow_costs(const uint32_t* c1, const uint32_t* c2, int W, int H, int K, int KP, int u1_min, int u2_min,
                       int oob, uint8_t* D1, uint8_t* D2, cudaStream_t s);
// Longest leaf block of the packed pair kernels (nodes); the V tensor maps'
// leaf boxes have this many rows.  Overridable for experiments.
#ifndef DMM_CMAX
#define DMM_CMAX 12
#endif
constexpr int kLeafMax = DMM_CMAX;

// Device-side bounds / invariant checks (assert) for a checking build
// (DMM_NVCC_EXTRA=-DDMM_DEVICE_CHECKS; compute-sanitizer is not available on
// the GPU pool): staging counts, stack depths, task ranges, shared indices.
#ifdef DMM_DEVICE_CHECKS
#include <cassert>
#define DMM_CHECK(c) assert(c)
#else
#define DMM_CHECK(c) ((void)0)
#endif

// Encode the V tensor maps of one frame (tmap.cu) into dev (4 x 128 B):
// records `fv` [H][W] of rec bytes, cost volume D [H][W][KP]; box rows 16 / 8 /
// 12 / 12.  Returns cudaSuccess or the error of the encode / copy.
constexpr int kTmapBytes = 4 * 128;
cudaError_t build_vmaps(uint8_t* fv, uint8_t* D, int W, int H, int KP, uint8_t* dev);
void launch_energy(const Layout& L, int frame0, int nframes, int w_h, int w_v, int T, int fbits,
                   const uint8_t* labels, int32_t* bad, cudaStream_t s);
void launch_unpad_u8(const uint8_t* src, uint8_t* dst, long long cells, int K, int KP, cudaStream_t s);
// dense u8 [cells][K] -> padded [cells][KP] (pads = 0)
void launch_pad_u8(const uint8_t* src, uint8_t* dst, long long cells, int K, int KP, cudaStream_t s);
// Expand compact records to dense int32 [cells][K]; if D != nullptr subtract
// D*2^fbits (recovers g_ from fh).
// Dense int32 [cells][KP] duals (general model) -> dense [cells][K], minus D*2^F if D.
void launch_decode_dense(const int32_t* src, const uint8_t* D, int fbits, int32_t* dst, long long cells, int K, int KP,
                         cudaStream_t s);
void launch_decode_rec(const uint8_t* rec, const uint8_t* D, int fbits, int32_t* dst, long long cells, int K,
                       int KP, cudaStream_t s);

}  // namespace dmm
