// hm_impl.cuh -- Dual MM half-steps (Algorithm 2) for sm_100a: every row
// (H pass) or column (V pass) chain builds its hierarchical minorant
// with Handshakes (Alg.5).
//
// One chain per warp in int32: the fallback of the packed chain-pair kernels
// (hm2.cu) for configurations outside their 16-bit range check, and the
// DMM_TUNE_PAIR = 0 path.  Mapping:
//  * a warp owns one K-vector at a time with the label dimension in registers,
//    LPL = KP/32 consecutive labels per lane; Msg / Handshake are the
//    register-level primitives of hm_device.cuh.
//  * node data F (the pass's unaries: D*2^F + g_ for H, f_ for V) are compact
//    u16-span records (dmm_internal.cuh); they stream into a per-warp ring of
//    kNSlot chunks x kCH nodes filled by TMA bulk copies (cp.async.bulk, one
//    mbarrier per chunk); full chunks run unrolled with compile-time offsets.
//  * level-synchronous launches: the root (level 0, two warps per chain: the
//    forward and the backward pass, then the Handshake), the global levels
//    1..l*-1 (one warp per (chain, subchain) task; only the message direction
//    whose boundary changed is recomputed -- Fig.11's reuse: "spine" messages
//    a later level needs go to the fwd/bwd scratch arrays), and the leaf blocks.
//  * leaf blocks (the 2^l* subchains of length <= kCMax), one warp per block:
//    TMA stages the block's records, D rows and its two boundary messages, and
//    the warp finishes the sub-hierarchy on chip, depth first, the forward and
//    backward passes of each piece interleaved (two independent Msg chains ->
//    ILP), pending pieces on a compact-record stack.  A leaf [p,p] with
//    boundary messages L, R has lambda = L + F + R (reading R8); the pass
//    writes L + R + D*2^F, which is f_ = lambda - g_ for H and D*2^F + g_ (the
//    next H pass's unaries) for V, as a compact record.  Node minima of lambda
//    sum to the dual bound (exactness); the last V pass writes the
//    lowest-index argmin as the label (R13, R14).
// All arithmetic is exact int32 (ranges in DESIGN.md): bit-identical to the
// CPU oracle whatever the evaluation order.
#pragma once
#include "hm_device.cuh"

namespace dmm {

constexpr int kCMax = 12;    // longest leaf block (nodes); < 16 (4-bit piece starts)
constexpr int kDepth = 4;    // pending right pieces in a leaf block (ceil(log2 kCMax))
constexpr int kNWG = 8;      // warps per CTA, level kernels
constexpr int kNWL = 8;      // warps per CTA, leaf kernel

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

// [lo, hi] of subchain s (bit-path from the root, MSB first) at level lev.
__device__ __forceinline__ void task_bounds(int n, int lev, int s, int& lo, int& hi) {
    lo = 0; hi = n - 1;
    for (int b = lev - 1; b >= 0; --b) {
        const int mid = lo + (hi - lo + 1) / 2 - 1;
        if ((s >> b) & 1) lo = mid + 1; else hi = mid;
    }
}

// Per-pass constants shared by both kernels.
template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
struct Pass {
    static constexpr int KP = 32 * LPL;
    static constexpr int REC = rec_bytes(KP);
    static constexpr int SREC = FIRST ? KP : REC;   // bytes of a source record (FIRST: the D row)
    FramePtrs P;
    const uint8_t* src;     // source records: FIRST ? D : (VERT ? fv : fh)
    uint8_t* dst;           // output records: VERT ? fh : fv
    int W, K, c, lane, n;
    int fbits, ws, wsT;

    __device__ __forceinline__ void init(const PassArgs& a, int chain, int lane_) {
        P = frame_ptrs(a.L, a.frame0 + blockIdx.y);
        src = FIRST ? P.D : (VERT ? P.fv : P.fh);
        dst = VERT ? P.fh : P.fv;
        W = a.L.W; K = a.L.K; c = chain; lane = lane_;
        n = VERT ? a.L.H : a.L.W;
        fbits = a.fbits; ws = a.ws; wsT = a.wsT;
    }
    __device__ __forceinline__ int q_of(int p) const { return VERT ? p * W + c : c * W + p; }
    __device__ __forceinline__ size_t moff(int p) const { return (size_t)q_of(p) * KP + lane * LPL; }
    __device__ __forceinline__ void msg_(int (&x)[LPL]) const { msg<LPL, PAD, WIN>(x, ws, wsT, lane, K); }
    // decode a staged source record at shared address `rec`: F (FIRST: D*2^F)
    __device__ __forceinline__ void dec(unsigned rec, int (&F)[LPL]) const {
        if constexpr (FIRST) {
            ld_u8_s<LPL>(rec + lane * LPL, F);
#pragma unroll
            for (int e = 0; e < LPL; ++e) F[e] <<= fbits;
        } else {
            ld_rec_s<LPL>(rec, lane, F);
        }
    }
};

// ============================================================ level kernels
// Global levels (subchains longer than kCMax) run level-synchronously: one
// launch per hierarchy level, one warp per (chain, subchain) task, no CTA
// barriers (the launch boundary orders the levels).  A task runs one pass --
// the direction whose boundary changed -- and the Handshake; the node records
// stream through a per-warp TMA ring.
template <int CH, int NS>
struct RingShared {     // per-warp shared memory (bytes): NS chunks of CH records
    int slot, ring, mbar, total;
    __host__ __device__ RingShared(int KP) {
        slot = CH * rec_bytes(KP);
        ring = 0;
        mbar = align_up(ring + NS * slot, 8);
        total = align_up(mbar + NS * 8, 128);
    }
};
// ring geometry: the root's two passes per chain are the latency-critical path
// with few warps per SM, so they prefetch deepest (64 nodes)
constexpr int kRootCH = 16, kRootNS = 4;
constexpr int kLevCH = 8, kLevNS = 4;

template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST, int kCH, int kNSlot>
struct Task : Pass<LPL, VERT, PAD, WIN, FIRST> {
    using B = Pass<LPL, VERT, PAD, WIN, FIRST>;
    using B::KP; using B::REC; using B::SREC;
    unsigned ring;                  // shared address of the ring
    unsigned mbar;                  // shared address of the NS mbarriers (8 B each)
    int slotB;
    // the task's runs: 0 = its pass, 1 = the Handshake pair (j, i) (absent for the root's bwd warp)
    int rs0, rd0, rc0, rs1, rd1, rc1, nruns, cur;
    int r_start, r_dir, r_left;     // producer: rest of the current run
    unsigned long long clen;        // chunk length of slot s in bits 8s..8s+7 (per-lane copy)
    int cslot, cidx, ccount;        // consumer position
    bool crev;                      // current chunk holds a descending run
    unsigned cphase;                // consumer parity bit per slot (kept across tasks)
    bool cwait;

    __device__ __forceinline__ void fill(int slot) {
        while (r_left == 0) {
            if (cur >= nruns) return;
            if (cur == 0) { r_start = rs0; r_dir = rd0; r_left = rc0; }
            else { r_start = rs1; r_dir = rd1; r_left = rc1; }
            ++cur;
        }
        const int cnt = r_left < kCH ? r_left : kCH;
        const unsigned sbase = ring + slot * slotB;
        const unsigned bar = mbar + 8 * slot;
        // slot holds the chunk's records at stride SREC in ascending node order;
        // bit 7 of the chunk's byte marks a descending run
        const unsigned long long rev = (!VERT && r_dir < 0) ? 0x80ull : 0ull;
        clen = (clen & ~(0xffull << (8 * slot))) | (((unsigned long long)cnt | rev) << (8 * slot));
        if (this->lane == 0) mbar_expect_tx_s(bar, (unsigned)(cnt * SREC));
        __syncwarp();
        fence_proxy_async();     // the slot was read through the generic proxy
        __syncwarp();
        if constexpr (!VERT) {   // H: the chunk's records are contiguous -> one bulk copy
            if (this->lane == 0) {
                const int first = r_dir > 0 ? r_start : r_start - cnt + 1;
                tma_load_s(sbase, this->src + (size_t)this->q_of(first) * SREC, cnt * SREC, bar);
            }
        } else if (this->lane < cnt) {
            const size_t q = (size_t)this->q_of(r_start + r_dir * this->lane);
            tma_load_s(sbase + this->lane * SREC, this->src + q * SREC, SREC, bar);
        }
        r_start += r_dir * cnt;
        r_left -= cnt;
    }
    __device__ __forceinline__ void ring_init(char* wsm, const RingShared<kCH, kNSlot>& lay) {
        ring = smem_addr(wsm + lay.ring);
        mbar = smem_addr(wsm + lay.mbar);
        slotB = lay.slot;
        if (this->lane == 0) {
            uint64_t* b = reinterpret_cast<uint64_t*>(wsm + lay.mbar);
            for (int k = 0; k < kNSlot; ++k) mbar_init(&b[k], 1);
            fence_mbar_init();
        }
        __syncwarp();
        cphase = 0;
    }
    // start streaming a task's runs (the previous task's chunks are all consumed)
    __device__ __forceinline__ void start(int nr) {
        nruns = nr; cur = 0; r_left = 0; clen = 0;
        cslot = 0; cidx = 0; ccount = 0; cwait = true;
        for (int k = 0; k < kNSlot; ++k) fill(k);
    }
    __device__ __forceinline__ void chunk_wait() {
        mbar_wait_s(mbar + 8 * cslot, (cphase >> cslot) & 1u);
        __syncwarp();
        cphase ^= 1u << cslot;
        const unsigned b = (unsigned)((clen >> (8 * cslot)) & 0xffull);
        ccount = (int)(b & 0x7fu);
        crev = (b & 0x80u) != 0;
        cidx = 0;
        cwait = false;
    }
    __device__ __forceinline__ void chunk_release() {
        __syncwarp();
        fill(cslot);
        cslot = cslot + 1 == kNSlot ? 0 : cslot + 1;
        cwait = true;
    }
    __device__ __forceinline__ void pop(int (&F)[LPL]) {
        if (cwait) chunk_wait();
        this->dec(ring + cslot * slotB + (crev ? ccount - 1 - cidx : cidx) * SREC, F);
        if (++cidx == ccount) chunk_release();
    }
    // ---- passes: DIR = +1 forward from `first` (phi_{p+1} = Msg(phi_p + F_p)),
    // DIR = -1 backward; nsteps Msgs.  Spine messages a later level needs go to
    // the fwd/bwd scratch arrays: forward over a piece of len0 = nsteps + 1
    // nodes, nodes first + (len0 >> k) - 1; backward, first - ceil(len0/2^k) + 1.
    // The pass is run 0 of the task, so its chunks hold exactly its nodes; full
    // chunks run unrolled with compile-time ring offsets.
    template <int DIR>
    __device__ __forceinline__ void run_pass(int first, int nsteps, int (&phi)[LPL]) {
        if (nsteps < 1) return;
        constexpr bool REV = !VERT && DIR < 0;   // H backward chunks are staged ascending
        const int len0 = nsteps + 1;
        int kk = DIR > 0 ? (31 - __clz(len0)) - 1 : 31 - __clz(len0 - 1);
        int target = DIR > 0 ? (len0 >> kk) : (((len0 - 1) >> kk) + 1);
        int32_t* arr = DIR > 0 ? this->P.fwd : this->P.bwd;
        auto spine = [&](int s) {
            if (s + 2 == target) {
                st_i32<LPL>(arr + this->moff(first + DIR * (s + 1)), phi);
                --kk;
                target = kk < 0 ? INT_MAX : (DIR > 0 ? (len0 >> kk) : (((len0 - 1) >> kk) + 1));
            }
        };
        int s = 0;
#pragma unroll 1
        while (s < nsteps) {
            chunk_wait();
            const unsigned base = ring + cslot * slotB;
            if (ccount == kCH) {
                int F[LPL];
                this->dec(base + (REV ? kCH - 1 : 0) * SREC, F);
#pragma unroll
                for (int k = 0; k < kCH; ++k) {
#pragma unroll
                    for (int e = 0; e < LPL; ++e) phi[e] += F[e];
                    if (k + 1 < kCH) this->dec(base + (REV ? kCH - 2 - k : k + 1) * SREC, F);
                    this->msg_(phi);
                    spine(s + k);
                }
                s += kCH;
            } else {
                const int cnt = ccount;
                int F[LPL];
                this->dec(base + (REV ? cnt - 1 : 0) * SREC, F);
#pragma unroll 1
                for (int k = 0; k < cnt; ++k) {
#pragma unroll
                    for (int e = 0; e < LPL; ++e) phi[e] += F[e];
                    if (k + 1 < cnt) this->dec(base + (REV ? cnt - 2 - k : k + 1) * SREC, F);
                    this->msg_(phi);
                    spine(s + k);
                }
                s += cnt;
            }
            chunk_release();
        }
    }
    // Handshake (Alg.5); the ring delivers F_j then F_i.  Writes the
    // children's new boundaries: fwd[j] = phi_ij, bwd[i] = phi_ji'.
    __device__ __forceinline__ void handshake(int i, int (&pl)[LPL], int (&pr)[LPL]) {
        int Fi[LPL], Fj[LPL];
        pop(Fj);
        pop(Fi);
        handshake_regs<LPL, PAD, WIN>(Fi, Fj, pl, pr, this->ws, this->wsT, this->lane, this->K);
        st_i32<LPL>(this->P.fwd + this->moff(i + 1), pl);
        st_i32<LPL>(this->P.bwd + this->moff(i), pr);
    }
};

// Level 0: the whole chain [0, n-1] with zero boundary messages; warp 0 runs the
// forward pass into i, warp 1 the backward pass into j, warp 0 the Handshake.
template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
__global__ void __launch_bounds__(64) hm_root_kernel(PassArgs a) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int KP = 32 * LPL;
    const RingShared<kRootCH, kRootNS> lay(KP);
    Task<LPL, VERT, PAD, WIN, FIRST, kRootCH, kRootNS> h;
    h.init(a, blockIdx.x, lane);
    h.ring_init(smem + warp * lay.total, lay);
    const int n = h.n, i = n / 2 - 1, j = i + 1;
    int zero[LPL], phi[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) { zero[e] = 0; phi[e] = 0; }
    if (warp == 0) {
        h.rs0 = 0; h.rd0 = 1; h.rc0 = i;
        h.rs1 = j; h.rd1 = -1; h.rc1 = 2;
        h.start(2);
        st_i32<LPL>(h.P.fwd + h.moff(0), zero);
        h.template run_pass<1>(0, i, phi);
    } else {
        h.rs0 = n - 1; h.rd0 = -1; h.rc0 = n - 1 - j;
        h.start(1);
        st_i32<LPL>(h.P.bwd + h.moff(n - 1), zero);
        h.template run_pass<-1>(n - 1, n - 1 - j, phi);
        st_i32<LPL>(h.P.bwd + h.moff(j), phi);
    }
    __syncthreads();
    if (warp == 0) {
        int pr[LPL];
        ld_i32<LPL>(h.P.bwd + h.moff(j), pr);
        h.handshake(i, phi, pr);
    }
}

// Level lev >= 1: one warp per (chain, subchain s) task.
template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST, int NW>
__global__ void __launch_bounds__(NW * 32) hm_level_kernel(PassArgs a, int lev, int ntasks) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int KP = 32 * LPL;
    const RingShared<kLevCH, kLevNS> lay(KP);
    Task<LPL, VERT, PAD, WIN, FIRST, kLevCH, kLevNS> h;
    h.init(a, 0, lane);
    h.ring_init(smem + warp * lay.total, lay);
    const int n = h.n;
#pragma unroll 1
    for (int t = blockIdx.x * NW + warp; t < ntasks; t += gridDim.x * NW) {
        h.c = t >> lev;
        const int s = t & ((1 << lev) - 1);
        int lo, hi;
        task_bounds(n, lev, s, lo, hi);
        const int ii = lo + (hi - lo + 1) / 2 - 1, j = ii + 1;
        int bnd[LPL], spn[LPL];
        if (!(s & 1)) {   // left piece: left boundary kept -> reuse fwd, recompute bwd
            h.rs0 = hi; h.rd0 = -1; h.rc0 = hi - j;
            h.rs1 = j; h.rd1 = -1; h.rc1 = 2;
            h.start(2);
            ld_i32<LPL>(h.P.bwd + h.moff(hi), bnd);
            ld_i32<LPL>(h.P.fwd + h.moff(ii), spn);
            h.template run_pass<-1>(hi, hi - j, bnd);
            h.handshake(ii, spn, bnd);
        } else {          // right piece: right boundary kept -> reuse bwd, recompute fwd
            h.rs0 = lo; h.rd0 = 1; h.rc0 = ii - lo;
            h.rs1 = j; h.rd1 = -1; h.rc1 = 2;
            h.start(2);
            ld_i32<LPL>(h.P.fwd + h.moff(lo), bnd);
            ld_i32<LPL>(h.P.bwd + h.moff(j), spn);
            h.template run_pass<1>(lo, ii - lo, bnd);
            h.handshake(ii, bnd, spn);
        }
    }
}

// ============================================================== leaf kernel
struct LeafShared {     // per-warp shared memory (bytes)
    int L, R, F, D, stack, mbar, total;
    __host__ __device__ LeafShared(int KP) {
        const int rec = rec_bytes(KP);
        L = 0;
        R = L + KP * 4;
        F = R + KP * 4;                 // kCMax source records (stride REC)
        D = F + kCMax * rec;            // kCMax D rows
        stack = D + kCMax * KP;         // kDepth x (phi_ij, R) compact records
        mbar = align_up(stack + kDepth * 2 * rec, 8);
        total = align_up(mbar + 8, 128);
    }
};

// Emit leaf `node` (chain index) with boundary messages Lb, Rb, unaries F and
// its staged D row at shared address dD: lambda = L + F + R (reading R8); the
// output record is L + R + D*2^F; bound += min lambda; last V: label.
template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
__device__ __forceinline__ void leaf_emit(const Pass<LPL, VERT, PAD, WIN, FIRST>& h, unsigned dD, int node,
                                          const int (&Lb)[LPL], const int (&Rb)[LPL], const int (&F)[LPL],
                                          bool last, long long& bsum) {
    constexpr int REC = Pass<LPL, VERT, PAD, WIN, FIRST>::REC;
    const int lane = h.lane;
    int Dv[LPL], lam[LPL], o[LPL];
    ld_u8_s<LPL>(dD + lane * LPL, Dv);
    int lmin = INT_MAX;
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        const int lr = Lb[e] + Rb[e];
        o[e] = lr + (Dv[e] << h.fbits);
        lam[e] = lr + F[e];
        if (PAD && lane * LPL + e >= h.K) lam[e] = INT_MAX;
        lmin = min(lmin, lam[e]);
    }
    const int q = h.q_of(node);
    st_rec<LPL, PAD>(h.dst + (size_t)q * REC, lane, o, h.K);
    const int gmin = __reduce_min_sync(kFull, lmin);
    bsum += gmin;
    if (VERT && last) {
        int kmin = INT_MAX;
#pragma unroll
        for (int e = LPL - 1; e >= 0; --e)
            if (lam[e] == gmin) kmin = lane * LPL + e;
        kmin = __reduce_min_sync(kFull, kmin);
        if (lane == 0) h.P.labels[q] = (uint8_t)kmin;
    }
}

// One warp per leaf block [lo, hi] (level lstar): TMA-stage its records, D rows
// and boundary messages, then solve its sub-hierarchy on chip, depth first.
template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
__global__ void __launch_bounds__(kNWL * 32) hm_leaf_kernel(PassArgs a, int lstar, int nblocks) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    using PS = Pass<LPL, VERT, PAD, WIN, FIRST>;
    constexpr int KP = PS::KP, REC = PS::REC, SREC = PS::SREC;
    const LeafShared lay(KP);
    char* wsm = smem + warp * lay.total;
    const unsigned wsa = smem_addr(wsm);
    const unsigned sF = wsa + lay.F;
    const unsigned sD = FIRST ? sF : wsa + lay.D;
    const int strideD = KP;                    // FIRST: the D rows are the staged records (SREC = KP)
    uint8_t* stk = reinterpret_cast<uint8_t*>(wsm + lay.stack);
    const unsigned bar = wsa + lay.mbar;
    if (lane == 0) { mbar_init(reinterpret_cast<uint64_t*>(wsm + lay.mbar), 1); fence_mbar_init(); }
    __syncwarp();
    unsigned phase = 0;
    const bool last = a.last != 0;
    const int nbl = 1 << lstar;
    long long bsum = 0;
    PS h;
    h.init(a, 0, lane);
    const int n = h.n;

#pragma unroll 1
    for (int b = blockIdx.x * kNWL + warp; b < nblocks; b += gridDim.x * kNWL) {
        h.c = b >> lstar;
        int lo0, hi0;
        task_bounds(n, lstar, b & (nbl - 1), lo0, hi0);
        const int m = hi0 - lo0 + 1;
        // ---- stage: records, D rows, boundary messages (one mbarrier phase)
        const unsigned bytes = m * SREC + (FIRST ? 0 : m * KP) + (lstar > 0 ? 2 * KP * 4 : 0);
        if (lane == 0) mbar_expect_tx_s(bar, bytes);
        __syncwarp();
        fence_proxy_async();
        __syncwarp();
        if constexpr (!VERT) {   // H: the block's records and D rows are contiguous
            if (lane == 0) {
                const size_t q = (size_t)h.q_of(lo0);
                tma_load_s(sF, h.src + q * SREC, m * SREC, bar);
                if (!FIRST) tma_load_s(sD, h.P.D + q * KP, m * KP, bar);
            }
        } else if (lane < m) {
            const size_t q = (size_t)h.q_of(lo0 + lane);
            tma_load_s(sF + lane * SREC, h.src + q * SREC, SREC, bar);
            if (!FIRST) tma_load_s(sD + lane * KP, h.P.D + q * KP, KP, bar);
        }
        if (lstar > 0 && lane == 30)
            tma_load_s(wsa + lay.L, h.P.fwd + (size_t)h.q_of(lo0) * KP, KP * 4, bar);
        if (lstar > 0 && lane == 31)
            tma_load_s(wsa + lay.R, h.P.bwd + (size_t)h.q_of(hi0) * KP, KP * 4, bar);
        mbar_wait_s(bar, phase);
        __syncwarp();
        phase ^= 1u;
        int L[LPL], R[LPL];
        if (lstar > 0) {
            ld_i32<LPL>(reinterpret_cast<const int32_t*>(wsm + lay.L) + lane * LPL, L);
            ld_i32<LPL>(reinterpret_cast<const int32_t*>(wsm + lay.R) + lane * LPL, R);
        } else {
#pragma unroll
            for (int e = 0; e < LPL; ++e) { L[e] = 0; R[e] = 0; }
        }
        // ---- the block's sub-hierarchy, depth first.  A child of length 1 is
        // emitted right after its parent's Handshake (its F is in registers) and
        // the walk continues with the sibling, so only pieces whose children
        // are both longer than one node push to the stack.
        int lo = 0, hi = m - 1, sp = 0;
        unsigned stkJ = 0, stkH = 0;   // pending pieces [j_k, hi_k], 4 bits each, per-lane registers
#pragma unroll 1
        while (true) {
            bool done_piece = false;
            if (lo == hi) {                       // a one-node block
                int F[LPL];
                h.dec(sF + lo * SREC, F);
                leaf_emit<LPL, VERT, PAD, WIN, FIRST>(h, sD + lo * strideD, lo0 + lo, L, R, F, last, bsum);
                done_piece = true;
            } else {
                const int len = hi - lo + 1, i = lo + len / 2 - 1, j = i + 1;
                int pl[LPL], pr[LPL];
#pragma unroll
                for (int e = 0; e < LPL; ++e) { pl[e] = L[e]; pr[e] = R[e]; }
                const int nf = i - lo, nb = hi - j;
#pragma unroll 1
                for (int s = 0; s < nf || s < nb; ++s) {
                    if (s < nf) {
                        int F[LPL];
                        h.dec(sF + (lo + s) * SREC, F);
#pragma unroll
                        for (int e = 0; e < LPL; ++e) pl[e] += F[e];
                        h.msg_(pl);
                    }
                    if (s < nb) {
                        int F[LPL];
                        h.dec(sF + (hi - s) * SREC, F);
#pragma unroll
                        for (int e = 0; e < LPL; ++e) pr[e] += F[e];
                        h.msg_(pr);
                    }
                }
                int Fi[LPL], Fj[LPL];
                h.dec(sF + i * SREC, Fi);
                h.dec(sF + j * SREC, Fj);
                handshake_regs<LPL, PAD, WIN>(Fi, Fj, pl, pr, h.ws, h.wsT, lane, h.K);
                // children: A = (lo, i, L, phi_ji' = pr), B = (j, hi, phi_ij = pl, R)
                const bool leafA = (i == lo), leafB = (j == hi);
                if (leafA) leaf_emit<LPL, VERT, PAD, WIN, FIRST>(h, sD + i * strideD, lo0 + i, L, pr, Fi, last, bsum);
                if (leafB) leaf_emit<LPL, VERT, PAD, WIN, FIRST>(h, sD + j * strideD, lo0 + j, pl, R, Fj, last, bsum);
                if (leafA && leafB) {
                    done_piece = true;
                } else if (leafA) {                 // continue with B
                    lo = j;
#pragma unroll
                    for (int e = 0; e < LPL; ++e) L[e] = pl[e];
                } else if (leafB) {                 // continue with A
                    hi = i;
#pragma unroll
                    for (int e = 0; e < LPL; ++e) R[e] = pr[e];
                } else {                            // push B, continue with A
                    stkJ = (stkJ & ~(0xfu << (4 * sp))) | ((unsigned)j << (4 * sp));
                    stkH = (stkH & ~(0xfu << (4 * sp))) | ((unsigned)hi << (4 * sp));
                    __syncwarp();   // every lane has read this stack slot's previous bases
                    st_rec<LPL, false>(stk + (2 * sp) * REC, lane, pl, h.K);
                    st_rec<LPL, false>(stk + (2 * sp + 1) * REC, lane, R, h.K);
                    ++sp;
                    hi = i;
#pragma unroll
                    for (int e = 0; e < LPL; ++e) R[e] = pr[e];
                }
            }
            if (done_piece) {
                if (sp == 0) break;
                --sp;
                lo = (int)((stkJ >> (4 * sp)) & 0xfu);
                hi = (int)((stkH >> (4 * sp)) & 0xfu);
                __syncwarp();   // record bases were written by lane 0
                ld_rec<LPL>(stk + (2 * sp) * REC, lane, L);
                ld_rec<LPL>(stk + (2 * sp + 1) * REC, lane, R);
            }
        }
        __syncwarp();   // all lanes done with the staged block before the next fill
    }
    if (lane == 0 && bsum != 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&h.P.bounds[a.bound_slot]), (unsigned long long)bsum);
}

// ================================================================ launchers
// Leaf level: smallest l with ceil(n / 2^l) <= kCMax.
static int leaf_level(int n) {
    int l = 0;
    while (((n + (1 << l) - 1) >> l) > kCMax) ++l;
    return l;
}

// Per-instantiation launch constants (SM count, occupancy, smem opt-in),
// queried once per device: host API calls between the ~8 launches of a
// half-step would otherwise starve the GPU.
struct LaunchCache {
    int dev = -1, sms = 148, lev_cap = 148, leaf_cap = 148;
};

template <int LPL, bool PAD, int WIN, bool FIRST, bool VERT>
static void launch_cfg(const PassArgs& a, int nframes, cudaStream_t s) {
    constexpr int KP = 32 * LPL;
        const int chains = VERT ? a.L.W : a.L.H;
    const int units = chains;
    const int n = VERT ? a.L.H : a.L.W;
    const int lstar = leaf_level(n);
    const int rr = RingShared<kRootCH, kRootNS>(KP).total;
    const int rs = RingShared<kLevCH, kLevNS>(KP).total;
    const int smem = kNWL * LeafShared(KP).total;
    auto rk = hm_root_kernel<LPL, VERT, PAD, WIN, FIRST>;
    auto lk = hm_level_kernel<LPL, VERT, PAD, WIN, FIRST, kNWG>;
    auto kern = hm_leaf_kernel<LPL, VERT, PAD, WIN, FIRST>;
    static LaunchCache lc;
    int dev = 0;
    cudaGetDevice(&dev);
    if (lc.dev != dev) {
        cudaDeviceGetAttribute(&lc.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * rr);
        cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, kNWG * rs);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lk, kNWG * 32, kNWG * rs);
        lc.lev_cap = lc.sms * (per_sm > 0 ? per_sm : 1);
        per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNWL * 32, smem);
        lc.leaf_cap = lc.sms * (per_sm > 0 ? per_sm : 1);
        lc.dev = dev;
    }
    if (lstar > 0) {
        rk<<<dim3(units, nframes), 64, 2 * rr, s>>>(a);
        for (int lev = 1; lev < lstar; ++lev) {
            const int ntasks = units << lev;
            int grid = (ntasks + kNWG - 1) / kNWG;
            if (grid > lc.lev_cap) grid = lc.lev_cap;
            lk<<<dim3(grid, nframes), kNWG * 32, kNWG * rs, s>>>(a, lev, ntasks);
        }
    }
    const int nblocks = units << lstar;
    int grid = (nblocks + kNWL - 1) / kNWL;
    if (grid > lc.leaf_cap) grid = lc.leaf_cap;
    kern<<<dim3(grid, nframes), kNWL * 32, smem, s>>>(a, lstar, nblocks);
}

template <int LPL, bool PAD, int WIN>
static void launch_dir(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    if (vertical) launch_cfg<LPL, PAD, WIN, false, true>(a, nframes, s);
    else if (a.first) launch_cfg<LPL, PAD, WIN, true, false>(a, nframes, s);
    else launch_cfg<LPL, PAD, WIN, false, false>(a, nframes, s);
}

template <int LPL, bool PAD>
void hm_launch_win(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    if (a.T > LPL + 1) launch_dir<LPL, PAD, 0>(a, vertical, nframes, s);
    else if constexpr (LPL >= 4) {
        if (a.T == 4) launch_dir<LPL, PAD, 4>(a, vertical, nframes, s);   // the default T
        else launch_dir<LPL, PAD, -1>(a, vertical, nframes, s);
    } else {
        launch_dir<LPL, PAD, -1>(a, vertical, nframes, s);
    }
}

}  // namespace dmm
