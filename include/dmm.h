/*
 * dmm.h -- C ABI of the B200 (sm_100a) hot path of arXiv 1601.06274
 * (Shekhovtsov, Reinbacher, Graber, Pock, "Solving Dense Image Matching in
 * Real-Time using Discrete-Continuous Optimization", CVWW 2016):
 *
 *   census transform -> Hamming cost volume -> K iterations of Dual MM
 *   (Algorithm 2) with hierarchical (Handshake) minorants -> labelling,
 *   primal energy, dual bound.
 *
 * Citations "P:n" are lines of the paper text with the section /
 * equation / algorithm they fall in; readings of silent or garbled passages are
 * numbered R1..R21 in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - extern "C", never throw, return dmm_status (DMM_OK == 0).
 *  - Device pointers are CUDA global-memory pointers on the context's device;
 *    host pointers are ordinary (preferably pinned) host memory.
 *  - `stream` is a cudaStream_t passed as void*; NULL = legacy default stream.
 *    Every call is stream-ordered and asynchronous unless it says "synchronises".
 *  - Every entry point taking a context runs on the context's device and
 *    restores the caller's current CUDA device before returning.
 *  - Ownership: the caller owns images, outputs and the device workspace
 *    (allocate with dmm_workspace_bytes()); the context owns only small host
 *    state.  A context is single-threaded; distinct contexts are independent.
 *  - Integers are exact.  Costs, bounds and energies are int64 in units of
 *    2^-frac_bits (fixed point, reading R9); E(x) is an integer times 2^F.
 *  - Layouts: images / labels row-major [H][W] (u8); cost volume and duals are
 *    exported label-contiguous and dense: [H][W][K].
 *  - Errors: DMM_E_ARG invalid argument / config, DMM_E_SHAPE pitch < width,
 *    DMM_E_STATE solve before cost volume / result before solve,
 *    DMM_E_CUDA a CUDA runtime error (text in dmm_last_error()),
 *    DMM_E_NCCL an NCCL error of a sharded context (dmm_shard),
 *    DMM_E_RANGE config outside the exact compact-storage range (dmm_create).
 */
#ifndef DMM_B200_H
#define DMM_B200_H
#include <stddef.h>
#include <stdint.h>
#if defined(__GNUC__)
#define DMM_API __attribute__((visibility("default")))
#else
#define DMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DMM_OK = 0,
    DMM_E_ARG = 1,
    DMM_E_SHAPE = 2,
    DMM_E_STATE = 3,
    DMM_E_CUDA = 4,
    DMM_E_NCCL = 5,
    DMM_E_RANGE = 6
} dmm_status;

typedef struct dmm_config {
    int32_t width, height;   /* 1..16384 each; the grid of P:145-152 (4-connected)      */
    int32_t d_min, d_max;    /* disparity range; K = d_max - d_min + 1 in [1, 256]       */
    int32_t census_radius;   /* 1 (3x3, 8 bits) or 2 (5x5, 24 bits), R17         */
    int32_t w_h, w_v;        /* pairwise weights >= 0: f_ij = w * min(|a-b|, trunc)      */
    int32_t trunc;           /* T >= 1 (T = 1 is Potts); Fig.2 P:132-142 with eps = 1, R2 */
    int32_t frac_bits;       /* F in [0, 8]: fixed-point fractional bits (R9)            */
    int32_t oob_cost;        /* cost when x - d leaves the image; -1 => ((2r+1)^2-1)/2   */
    int32_t batch;           /* frames held by the context, >= 1 (C5 throughput mode)    */
    int32_t max_iters;       /* capacity of the per-frame bound history, >= 1            */
    /* General pairwise model (NEXT-3; all zero = the truncated-linear model
     * w * min(|a-b|, trunc) above).  Penalty in units of 2^-frac_bits:
     *   R(d) = min(pen_e1*min(d, pen_delta) + pen_e2*max(d - pen_delta, 0), pen_c)
     * (Fig.2 P:132-142 sampled at integer differences: slope eps = pen_e1/2^F
     * up to delta, slope pen_e2/2^F beyond, truncated at C = pen_c/2^F;
     * 0 <= pen_e1 <= pen_e2), and edge (i,j) of direction w (w_h / w_v) costs
     *   V_ij(d) = floor(w * om_ij * R(|d|) / 16),
     * om_ij = 16 (edge_weights = 0) or the edge-aware weight of the left image
     * (edge_weights = 1): om = clamp(round(16 exp(-5 |I_i - I_j| / 255)), 1, 16)
     * (Eq. regularizer-form; formula SPEC S:99, reading R30).
     * trunc is not used in this mode.  Runs the int32 general kernels (hmg.cu);
     * ROWCOL sharding is not available for it. */
    int32_t pen_e1, pen_e2, pen_delta, pen_c;
    int32_t edge_weights;
    /* Minorant of the chain subproblems (NEXT-4): 0 = hierarchical (Handshake,
     * P:809-856; the default, "used to obtain all visual experiments"), 1 =
     * iterative (Alg.4: iter_passes sweeps alternating direction,
     * lambda_i += floor(m_i / 2^iter_gshift), the last sweep with gamma = 1;
     * the paper's run max_pass = 3, gamma = 0.25 -> iter_passes 3, iter_gshift 2,
     * P:804).  The iterative minorant runs on the general int32 kernels (one
     * warp per chain, sequential along it). */
    int32_t minorant, iter_passes, iter_gshift;
} dmm_config;

typedef struct dmm_ctx dmm_ctx;

/* Bytes of device workspace a context with this config needs (0 if invalid). */
DMM_API size_t dmm_workspace_bytes(const dmm_config* cfg);

/* Bind a context to caller-owned device memory `workspace` (>= the size above,
 * 256-byte aligned) on CUDA device `device`.  *out receives the context.
 * The duals are stored as lossless u16-span records (DESIGN.md "Compact
 * duals"); configurations whose proven span bound
 *   (2 * max(w_h, w_v) * min(trunc, K-1) + max(census bits, oob)) * 2^frac_bits
 * exceeds 65535 are rejected with DMM_E_RANGE (e.g. defaults w=3, T=4, F=4,
 * 5x5 census: 768). */
DMM_API dmm_status dmm_create(const dmm_config* cfg, void* workspace, size_t bytes, int device,
                      dmm_ctx** out);
DMM_API void dmm_destroy(dmm_ctx* ctx);

/* Census codes of both images and the cost volume
 *   D[y][x][k] = popcount(cL(x,y) ^ cR(x - d_k, y)), d_k = d_min + k
 * (P:416 Hamming distance; P:161 f_i(x_i) = D_i(u(x_i)); R17, R18),
 * out-of-image samples = oob_cost.  left/right: device u8 images, row pitch
 * `pitch` bytes (>= width) of frame `frame`. */
DMM_API dmm_status dmm_cost_volume(dmm_ctx* ctx, int frame, const uint8_t* left, const uint8_t* right,
                           int64_t pitch, void* stream);

/* Dual MM (Algorithm 2): g_ := 0 (R4), then `iterations` times
 * H half-step (per row: h = HM(D*2^F + g_), f_ = h - g_) and V half-step (per
 * column: v = HM(f_), g_ = v - f_), HM = hierarchical minorant (P:809-856,
 * Handshake Alg.5).  The last V half-step writes the labelling
 * (lowest-index argmin of v, R13/R14) and every half step adds its dual bound
 * sum_chains min (Eq.7) to the history; finally the primal energy of
 * the labelling (Eq.3) is evaluated on the device.  Frames
 * [frame, frame+nframes) are solved in the same launches.
 * 1 <= iterations <= max_iters.  Asynchronous. */
DMM_API dmm_status dmm_solve(dmm_ctx* ctx, int frame, int nframes, int32_t iterations, void* stream);

/* Read back the primal energy of the labelling (Eq.3, scaled by 2^F)
 * and the dual bound b_{2K-1} plus the history b_0..b_{2K-1} (each nullable;
 * the history has 2*iterations entries).  Synchronises `stream`. */
DMM_API dmm_status dmm_result(dmm_ctx* ctx, int frame, int64_t* energy, int64_t* bound,
                      int64_t* bound_history, void* stream);

/* Device copy of the labelling: u8 [H][W] label indices (disparity = d_min + label). */
DMM_API dmm_status dmm_copy_labels(dmm_ctx* ctx, int frame, uint8_t* labels, void* stream);

/* Parity taps (device destinations): census codes (which 0 = left, 1 = right;
 * u32 [H][W]); cost volume u8 [H][W][K]; duals int32 [H][W][K] (which 0 = f_
 * after the last H half-step, 1 = g_ after the last V half-step). */
DMM_API dmm_status dmm_copy_codes(dmm_ctx* ctx, int frame, int which, uint32_t* dst, void* stream);
DMM_API dmm_status dmm_copy_cost_volume(dmm_ctx* ctx, int frame, uint8_t* dst, void* stream);
DMM_API dmm_status dmm_copy_dual(dmm_ctx* ctx, int frame, int which, int32_t* dst, void* stream);

/* End-to-end call with HOST buffers: copies both images host->device, runs
 * dmm_cost_volume + dmm_solve + energy, copies the labelling (u8 [H][W]) and
 * the scalars back.  Synchronises `stream`. */
DMM_API dmm_status dmm_run_host(dmm_ctx* ctx, int frame, const uint8_t* left_host,
                        const uint8_t* right_host, int32_t iterations, uint8_t* labels_host,
                        int64_t* energy, int64_t* bound, void* stream);

/* Batched forms for a stream of frames (BASELINE configs[4], throughput mode):
 * frames [frame, frame + nframes) in one launch per kernel.
 * dmm_cost_volume_frames: left/right device images stacked [nframes][height]
 *   rows of `pitch` bytes (pitch >= width); DMM_E_ARG / DMM_E_SHAPE as
 *   dmm_cost_volume, and frame ranges outside [0, batch).
 * dmm_run_host_frames: dmm_run_host for nframes frames: host images and
 *   labels stacked u8 [nframes][H][W]; energy[f], bound[f] (nframes entries
 *   each, scaled by 2^F).  Synchronises `stream`. */
DMM_API dmm_status dmm_cost_volume_frames(dmm_ctx* ctx, int frame, int nframes, const uint8_t* left,
                                          const uint8_t* right, int64_t pitch, void* stream);
DMM_API dmm_status dmm_run_host_frames(dmm_ctx* ctx, int frame, int nframes, const uint8_t* left_host,
                                       const uint8_t* right_host, int32_t iterations, uint8_t* labels_host,
                                       int64_t* energy, int64_t* bound, void* stream);

/* Continuous refinement of the frame's labelling (NEXT-2; Sec. 2.4 P:283-405,
 * Sec. 3.1): the non-convex primal-dual iterates (Eq.
 * cont_iterates P:306-311, Valkonen's PDHG on the DC split
 * r = r_{eps,delta} - r_{0,C+delta-eps*delta}, Eq. r-decompose P:364-375,
 * prox Eq. pprox) on the two-slope convex approximation of the
 * data term around the current solution, re-approximated
 * `warps` times with `iters` iterations each (5 x 40 in P:497).
 * Weights w_h / w_v of the config; float64 on the device (the oracle's precision;
 * u_out is rounded to float32).  Readings
 * R24-R28: h in label units, linear interpolation of D between
 * labels, tau * sigma * 8 < 1 for convergence (0.35 / 0.35 suggested).
 * eps = 1, C = trunc gives the discrete model's truncated-linear r.
 * u_out (nullable): device float [H][W], refined disparity (d_min + label
 * units).  energy (nullable, host): E(u) = D(u) + R(Au), double; if given the
 * call synchronises `stream`.  DMM_E_STATE before dmm_solve.  The iterations
 * of one warp are captured once into a CUDA graph (per frame and parameters)
 * and replayed. */
typedef struct dmm_refine_params {
    double eps, delta, C;     /* penalty r: slope eps up to delta, slope 1, truncated at C  */
    double h;                 /* data approximation step / trust region (labels)          */
    double tau, sigma;        /* primal / dual step sizes                                   */
    int32_t warps, iters;     /* re-approximations x PDHG iterations each                   */
} dmm_refine_params;
DMM_API dmm_status dmm_refine(dmm_ctx* ctx, int frame, const dmm_refine_params* prm, float* u_out, double* energy,
                              void* stream);

/* Continuous refinement of an optical flow field (NEXT-2; Sec. 3.2
 * P:449-467): u1 = d_min + labels of frame `frame`, u2 = v_min + labels of
 * frame `frame + 1` (after dmm_flow_cost_volume + dmm_solve of both layers)
 * refined with the regulariser of dmm_refine on each component and the data
 * term approximated by the quadratic of Eq. 19 (central-difference gradient
 * and full 2x2 Hessian of the census cost at the current flow, PSD part;
 * bilinear between integer displacements; readings R34-R36) with the joint
 * 2-D prox of Eq. 20 (both components iterate in lockstep).  float64 on the
 * device; u1_out / u2_out (nullable) device float [H][W] in pixels; energy
 * (nullable, host) = sum D(u) + R(Au1) + R(Au2), synchronises `stream` when
 * given.  Errors: DMM_E_ARG (bad frame / parameters), DMM_E_STATE (either
 * layer not solved, or a band-sharded context). */
DMM_API dmm_status dmm_flow_refine(dmm_ctx* ctx, int frame, int32_t v_min, const dmm_refine_params* prm,
                                   float* u1_out, float* u2_out, double* energy, void* stream);

/* Optical flow, discrete stage (NEXT-1; Eq. "flow decoupled costs"
 * P:163-170, Sec. 3.2): census codes of both images into frame
 * `frame`, then the optimistic decoupled costs of the 2-D label window
 *   D(a,b) = popcount(c1(x,y) ^ c2(x + u1(a), y + u2(b))) (oob outside the image),
 *   u1(a) = d_min + a (horizontal, the config's range), u2(b) = v_min + b (vertical),
 *   f1(a) = min_b D(a,b) -> cost volume of frame `frame`,
 *   f2(b) = min_a D(a,b) -> cost volume of frame `frame + 1`,
 * by one fused kernel that never stores the K*K volume.  Note the sign: flow
 * matches x + u (stereo matches x - d).  K = d_max - d_min + 1 must be 16, 32,
 * 48 or 64 (both layers have K labels); frames frame, frame+1 < batch.  The
 * two layers are then independent K-label problems ("two independent
 * stereo-like problems"): dmm_solve(ctx, frame, 2, ...) solves both
 * in the same launches; labels of frame / frame+1 are u1 - d_min / u2 - v_min. */
DMM_API dmm_status dmm_flow_cost_volume(dmm_ctx* ctx, int frame, const uint8_t* left, const uint8_t* right,
                                        int64_t pitch, int32_t v_min, void* stream);

/* ---- chain-DP primitives (no context; device int32 arrays, dense
 * [count][K], K in [1, 256], ws = w * 2^F >= 0, T >= 1).  They run exactly the
 * device code of the Dual MM kernels, one warp per K-vector.
 *
 * dmm_msg: message passing, Eq. msg-pass / Msg of Alg.5
 * for the truncated-linear f_ij (Fig.2 with eps = 1, reading R2):
 *   out[v][b] = min_a a[v][a] + ws * min(|a - b|, T).
 * dmm_handshake: Alg.5 (readings R9/R10) over one edge ij:
 *   phi_ji  = Msg(Fj + phiR);  m = phiL + Fi + phi_ji;
 *   phi_ij  = Msg(floor((m - 2 phi_ji) / 2));  phi_ji' = Msg(-phi_ij);
 * outputs phi_ij (into j) and phi_ji' (into i).  phiL = message into i from
 * the left, phiR = message into j from the right. */
DMM_API dmm_status dmm_msg(const int32_t* a, int32_t* out, int count, int K, int32_t ws, int32_t T,
                           void* stream);
DMM_API dmm_status dmm_handshake(const int32_t* Fi, const int32_t* Fj, const int32_t* phiL,
                                 const int32_t* phiR, int32_t* phi_ij, int32_t* phi_ji, int count,
                                 int K, int32_t ws, int32_t T, void* stream);

/* ---- building blocks for sharded solves (paper_1601_06274_b200/sharding.py)
 *
 * dmm_buffer_ptr: device address and size of one of a frame's arrays, and the
 * bytes per pixel: DMM_BUF_D (u8 [H][W][KP] cost volume, KP = padded K),
 * DMM_BUF_FV (records of f_, REC = 2*KP + 16 bytes per pixel, see DESIGN.md
 * "Compact duals"), DMM_BUF_FH (records of D*2^F + g_), DMM_BUF_LABELS
 * (u8 [H][W]), DMM_BUF_BOUNDS (int64 [2*max_iters]).
 * dmm_import_cost_volume: load a dense device cost volume u8 [H][W][K] (e.g. a
 * band sliced out of a full-frame context's dmm_copy_cost_volume) as the
 * frame's D; afterwards the frame is ready for dmm_half_step / dmm_solve.
 * dmm_half_step: one half-step of Algorithm 2 on frames
 * [frame, frame+nframes): vertical = 0 runs the H half-step of iteration t
 * (t = 0 reads D only: g_ = 0, reading R4), vertical = 1 the V half-step (on
 * t = iterations-1 it writes the labelling); bound slot 2t+vertical is reset
 * and accumulated.  The V half-step reads the FV records, the H half-step
 * (t > 0) the FH records, so a caller may exchange those between half-steps.
 * dmm_energy: primal energy (Eq.3, scaled by 2^F) of the frame's current
 * labels; synchronises `stream` and writes *energy.
 * dmm_energy_of: the same energy of an arbitrary labelling `labels` (device
 * u8 [H][W] label indices, disparity = d_min + label
 * energy_evaluate) against the frame's cost volume; DMM_E_STATE before the
 * cost volume, DMM_E_ARG if a label is >= K (checked on the device).
 * Synchronises `stream`. */
#define DMM_BUF_D 0
#define DMM_BUF_FV 1
#define DMM_BUF_FH 2
#define DMM_BUF_LABELS 3
#define DMM_BUF_BOUNDS 4
DMM_API dmm_status dmm_buffer_ptr(dmm_ctx* ctx, int frame, int which, void** ptr, size_t* bytes,
                                  int* bytes_per_pixel);
DMM_API dmm_status dmm_import_cost_volume(dmm_ctx* ctx, int frame, const uint8_t* D_dense, void* stream);
DMM_API dmm_status dmm_half_step(dmm_ctx* ctx, int frame, int nframes, int32_t t, int vertical,
                                 int32_t iterations, void* stream);
DMM_API dmm_status dmm_energy(dmm_ctx* ctx, int frame, int64_t* energy, void* stream);
DMM_API dmm_status dmm_energy_of(dmm_ctx* ctx, int frame, const uint8_t* labels, int64_t* energy, void* stream);

/* ---- multi-GPU sharding (one process per GPU)
 *
 * dmm_nccl_unique_id: a fresh NCCL communicator id (128 bytes) on the
 * calling rank (rank 0), to be broadcast to the other ranks by the caller
 * (e.g. torch.distributed).  NCCL is loaded at run time (libnccl.so.2: the
 * process's own, e.g. torch's, else the system's); DMM_E_NCCL if unavailable.
 *
 * dmm_shard(ctx, id, rank, world, mode) makes ctx rank `rank` of `world`:
 *  - DMM_SHARD_FRAMES: the caller gives every rank its own frames (contexts
 *    are independent, no data-path collective); only records rank/world and,
 *    if id != NULL, creates the communicator.
 *  - DMM_SHARD_ROWCOL: ONE frame (batch == 1) solved by all ranks.  Rank r
 *    owns rows [r*H/world .. ) for the H half-steps and columns [r*W/world ..)
 *    for the V half-steps (band sizes differ by <= 1; every column band
 *    >= 16 wide).  Chains of one orientation are independent, so the
 *    only exchange is the transpose of the dual records between half-steps:
 *    one grouped ncclSend / ncclRecv all-to-all per half-step, issued by the
 *    library on the call's stream; the bound history and energy are int64
 *    sums combined by ncclAllReduce and the labelling is all-gathered, so
 *    dmm_result / dmm_copy_labels / dmm_run_host return the whole frame's
 *    results on every rank, bit-identical to the unsharded solve.  Each rank
 *    computes the cost volume of its own row band and column band only.
 *    The context must have been created with the frame's full config and a
 *    workspace of >= dmm_shard_workspace_bytes(cfg, rank, world, mode)
 *    bytes (<= dmm_workspace_bytes for world >= 2); the packed chain-pair
 *    kernels must apply (DMM_TUNE_PAIR on, 16-bit range check) -- else DMM_E_ARG.
 *    dmm_shard with id == NULL creates no communicator ("external
 *    transport"): dmm_solve then returns DMM_E_STATE and the caller drives
 *    dmm_half_step and moves the bytes of dmm_shard_plan itself (tests).
 *    Full-frame parity taps (dmm_copy_cost_volume, dmm_copy_dual,
 *    dmm_buffer_ptr, dmm_import_cost_volume, dmm_energy_of, the *_frames
 *    calls) return DMM_E_STATE on a ROWCOL context.
 *  ncclCommInitRank is collective: every rank must call dmm_shard.
 *
 * Host-only (no device, no context; usable on CPU hosts):
 * dmm_shard_workspace_bytes: workspace a ROWCOL rank needs (0 if invalid).
 * dmm_shard_plan: the all-to-all of half-step `phase` (0: after H, f_
 *   records row band -> column band; 1: after V, D*2^F + g_ records back) as
 *   one dmm_xfer per peer (self included): byte ranges relative to the
 *   workspace base; returns the number of entries (= world; -1 on bad
 *   arguments), writes at most `max`.  Every range is contiguous.
 * dmm_shard_locate: byte offset (from the workspace base) of pixel (y, x)'s
 *   record / label in rank `rank`'s arrays (DMM_LOC_*), -1 if not owned. */
#define DMM_SHARD_FRAMES 0
#define DMM_SHARD_ROWCOL 1
#define DMM_LOC_FV_H 0     /* H band output records (f_), column segments */
#define DMM_LOC_FH_H 1     /* H band input records (D*2^F + g_)          */
#define DMM_LOC_FV_V 2     /* V band input records (f_)                  */
#define DMM_LOC_FH_V 3     /* V band output records (D*2^F + g_)         */
#define DMM_LOC_LABEL_V 4  /* V band labels (u8)                         */
#define DMM_LOC_BOUNDS 5   /* int64 bound history [2*max_iters] + energy  */
typedef struct dmm_xfer {
    int32_t peer;
    int64_t send_offset, send_bytes;   /* to peer   */
    int64_t recv_offset, recv_bytes;   /* from peer */
} dmm_xfer;
DMM_API dmm_status dmm_nccl_unique_id(uint8_t out[128]);
DMM_API dmm_status dmm_shard(dmm_ctx* ctx, const uint8_t* id, int rank, int world, int mode);
DMM_API size_t dmm_shard_workspace_bytes(const dmm_config* cfg, int rank, int world, int mode);
DMM_API int dmm_shard_plan(const dmm_config* cfg, int rank, int world, int phase, dmm_xfer* out, int max);
DMM_API int64_t dmm_shard_locate(const dmm_config* cfg, int rank, int world, int which, int y, int x);

/* Number of kernels this context has launched since creation. */
DMM_API int64_t dmm_launch_count(const dmm_ctx* ctx);

/* Per-kernel device timing with CUDA events recorded on the launching stream
 * around every kernel (enable != 0).  dmm_read_profile synchronises the
 * recorded events, writes per-class totals (ms[c], launches[c]) for the
 * classes c = 0 census, 1 cost volume, 2 H half-step, 3 V half-step,
 * 4 energy, 5 continuous refinement (arrays of DMM_PROFILE_CLASSES entries)
 * and clears the record. */
#define DMM_PROFILE_CLASSES 6
DMM_API dmm_status dmm_set_profiling(dmm_ctx* ctx, int enable);
DMM_API dmm_status dmm_read_profile(dmm_ctx* ctx, double* ms, int64_t* launches);

/* Tuning knobs (no effect on results, which are exact).
 * DMM_TUNE_DEBUG_STOP_AFTER_H (debug): value != 0 makes dmm_solve stop after
 * the first H half-step, for the parity tap of f_ after H_1 (dmm_copy_dual
 * which = 0).  Such a partial solve computes no energy and no labelling:
 * dmm_result, dmm_copy_labels and dmm_copy_dual(which = 1) return DMM_E_STATE. */
#define DMM_TUNE_DEBUG_STOP_AFTER_H 2
/* DMM_TUNE_PAIR: value != 0 (default) runs the half-steps on chain pairs in
 * packed 16-bit arithmetic (two chains per warp) whenever the configuration
 * passes the 16-bit range check (3*w*2^F*min(T,K) + 16*span bound + 4 <= 16383;
 * exact, identical results); 0 forces the one-chain int32 kernels. */
#define DMM_TUNE_PAIR 3
/* DMM_TUNE_QUERY_PAIR: sets dmm_last_error() to "pair" or "int32", the
 * kernel family the next half-step will use (value ignored). */
#define DMM_TUNE_QUERY_PAIR 4
DMM_API dmm_status dmm_set_tuning(dmm_ctx* ctx, int param, int64_t value);

DMM_API const char* dmm_status_str(dmm_status s);
DMM_API const char* dmm_last_error(const dmm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
