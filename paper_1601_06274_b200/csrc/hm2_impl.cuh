// hm2_impl.cuh -- Dual MM half-steps (Algorithm 2) on chain PAIRS: the
// packed-16-bit form of hm.cu.  Same hierarchy, schedule and results (exact
// integers, checked against the oracle); one warp advances two chains of the
// same orientation (rows 2r, 2r+1 or columns 2c, 2c+1) in the two halves of
// every register (hm2_device.cuh), which halves the ALU instructions per chain
// of every Msg.  An odd last chain is paired with itself (its B half is
// computed and dropped).  Used whenever the configuration passes the 16-bit
// range check (capi.cu pair_range_ok); otherwise hm.cu runs.
//
// Shared-memory staging per node: records of chain A and chain B.
//   H: a chunk / block holds the A run then the B run (two contiguous bulk
//      copies, stride SREC, B at +CH*SREC);
//   V: node k holds A then B (adjacent in HBM: q and q+1), stride 2*SREC.
// Spine messages (Fig.11 reuse, as in hm.cu) go to the fwd/bwd scratch as
// packed words at chain A's pixel, with the two offsets in fwdo/bwdo.
#pragma once
#include "hm2_device.cuh"

namespace dmm {
namespace p2 {

constexpr int kCMax = kLeafMax;              // longest leaf block (nodes)
constexpr int kDepth = kCMax > 12 ? 3 : 2;   // pending right pieces (pieces >= 4 nodes push; 12 -> 6 -> 3)
constexpr int kFB = kCMax > 15 ? 5 : 4;      // bits per packed piece start / end on the stack
static_assert(kCMax <= 24 && kDepth * kFB <= 32, "leaf stack");
// Tuning constants (overridable with -D for experiments; the defaults are the measured best)
#ifndef DMM_NWG
#define DMM_NWG 2
#endif
#ifndef DMM_NWL
#define DMM_NWL 4
#endif
#ifndef DMM_ROOT_CH
#define DMM_ROOT_CH 16
#endif
#ifndef DMM_LEV_CH
#define DMM_LEV_CH 8
#endif
#ifndef DMM_LEV_NS
#define DMM_LEV_NS 2
#endif
#ifndef DMM_LEAF_MINB
#define DMM_LEAF_MINB 1
#endif
template <int LPL> constexpr int nwg() { return DMM_NWG; }   // warps per CTA, level kernels: small CTAs spread the few tasks of the top levels over all SMs
constexpr int kNWL = DMM_NWL;      // warps per CTA, leaf kernel
constexpr int kRootCH = DMM_ROOT_CH, kRootNS = 2;
constexpr int kLevCH = DMM_LEV_CH, kLevNS = DMM_LEV_NS;
#ifndef DMM_LEV_MIN_CTAS
#define DMM_LEV_MIN_CTAS 12
#endif
constexpr int kLevMinCTAs = DMM_LEV_MIN_CTAS;   // 2-warp level CTAs per SM the register budget must allow
static_assert(kRootCH <= 16 && kLevCH <= 16, "pair_range_ok (capi.cu) allows 16 unnormalised steps");

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

// Programmatic dependent launch: the kernels of a half-step are launched with
// programmatic stream serialisation, so a kernel's prologue (ring / mbarrier
// setup and the TMA staging of the pass's node records, which were written
// before the half-step's root started) overlaps the tail of the previous
// level.  Everything that reads or writes the previous level's outputs (the
// spine scratch, bounds, labels, output records) comes after pdl_wait(),
// which returns once the previous kernel has completed and its writes are
// visible; pdl_trigger_late() lets the next kernel start its prologue.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Each CTA triggers its dependents when its own work is done: the next
// level's CTAs then launch into the SMs freed by the finishing CTAs and stage
// their records while the tail of this level runs, instead of taking SM
// resources (shared memory, registers) from CTAs that are still working.
// Measured against a trigger at the start of each CTA: C2 2.24 -> 2.13 ms,
// C3 12.3 -> 11.0 ms (11.3 ms without PDL).
__device__ __forceinline__ void pdl_trigger_late() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void task_bounds(int n, int lev, int s, int& lo, int& hi) {
    lo = 0; hi = n - 1;
    for (int b = lev - 1; b >= 0; --b) {
        const int mid = lo + (hi - lo + 1) / 2 - 1;
        if ((s >> b) & 1) lo = mid + 1; else hi = mid;
    }
}

template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
struct Pass {
    static constexpr int KP = 32 * LPL;
    static constexpr int REC = rec_bytes(KP);
    static constexpr int SREC = FIRST ? KP : REC;
    FramePtrs P;
    const uint8_t* src;
    uint8_t* dst;
    int W, K, cA, cB, lane, n, nch;
    bool hasB;
    int fbits, ws, wsT;
    DtK<LPL> dk;

    __device__ __forceinline__ void init(const PassArgs& a, int lane_) {
        P = frame_ptrs(a.L, a.frame0 + blockIdx.y);
        src = FIRST ? P.D : (VERT ? P.fv : P.fh);
        dst = VERT ? P.fh : P.fv;
        W = a.L.W; K = a.L.K; lane = lane_;
        n = VERT ? a.L.H : a.L.W;
        nch = VERT ? a.L.W : a.L.H;
        fbits = a.fbits; ws = a.ws; wsT = a.wsT;
        nseg = a.nseg; segx = a.segx; vtma = a.vtma;
        dk.init(ws, wsT, K, lane, a.T);
    }
    __device__ __forceinline__ void set_pair(int pc) {
        cA = 2 * pc;
        hasB = cA + 1 < nch;
        cB = hasB ? cA + 1 : cA;
    }
    int nseg;
    const int* segx;
    int vtma;
    __device__ __forceinline__ int q_of(int c, int p) const { return VERT ? p * W + c : c * W + p; }
    // record index of (chain c, position p) in the records the pass writes
    // (and, unless FIRST, reads): row-major, or column segments for H records
    // of a band-sharded context (PassArgs::segx)
    __device__ __forceinline__ size_t rq(int c, int p) const {
        if (VERT || nseg <= 1) return (size_t)q_of(c, p);
        int s = 0;
        while (p >= segx[s + 1]) ++s;
        const int x0 = segx[s], w = segx[s + 1] - x0;
        return (size_t)x0 * nch + (size_t)c * w + (p - x0);
    }
    __device__ __forceinline__ size_t srcq(int c, int p) const { return FIRST ? (size_t)q_of(c, p) : rq(c, p); }
    // number of records contiguous with (c, p) in a run of cnt ascending positions
    __device__ __forceinline__ int run1(int p, int cnt, bool segmented) const {
        if (VERT || nseg <= 1 || !segmented) return cnt;
        int s = 0;
        while (p >= segx[s + 1]) ++s;
        return min(cnt, segx[s + 1] - p);
    }
    __device__ __forceinline__ int qA(int p) const { return q_of(cA, p); }
    __device__ __forceinline__ int qB(int p) const { return q_of(cB, p); }
    __device__ __forceinline__ void msg_(unsigned (&x)[LPL], int& oa, int& ob) const {
        msg2<LPL, PAD, WIN>(x, oa, ob, dk);
    }
    // staged source pair (records, or D rows when FIRST) -> packed values + bases
    __device__ __forceinline__ void dec(unsigned ra, unsigned rb, unsigned (&v)[LPL], int& ba, int& bb) const {
        if constexpr (FIRST) {
            ld_u8_pair_s<LPL>(ra, rb, lane, fbits, v);
            ba = 0; bb = 0;
        } else {
            ld_rec_pair_s<LPL>(ra, rb, lane, v, ba, bb);
        }
    }
    __device__ __forceinline__ void st_spine(bool fwdarr, int p, const MP<LPL>& v) const {
        st_mp<LPL>(fwdarr ? P.fwd : P.bwd, fwdarr ? P.fwdo : P.bwdo, (size_t)qA(p), lane, v);
    }
    __device__ __forceinline__ void ld_spine(bool fwdarr, int p, MP<LPL>& v) const {
        ld_mp<LPL>(fwdarr ? P.fwd : P.bwd, fwdarr ? P.fwdo : P.bwdo, (size_t)qA(p), lane, v);
    }
};

// ============================================================ level kernels
template <int CH, int NS>
struct RingShared {     // per-warp shared memory (bytes): NS chunks of CH record pairs
    int slot, ring, mbar, total;
    __host__ __device__ RingShared(int KP, bool first) {
        slot = 2 * CH * (first ? KP : rec_bytes(KP));
        ring = 0;
        mbar = align_up(ring + NS * slot, 8);
        total = align_up(mbar + NS * 8, 128);
    }
};

template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST, int kCH, int kNSlot>
struct Task : Pass<LPL, VERT, PAD, WIN, FIRST> {
    using B = Pass<LPL, VERT, PAD, WIN, FIRST>;
    using B::KP; using B::REC; using B::SREC;
    static constexpr int kStride = VERT ? 2 * SREC : SREC;     // node stride inside a slot
    static constexpr int kOffB = VERT ? SREC : kCH * SREC;     // chain B's record, relative to A's
    unsigned ring, mbar;
    int slotB;
    int rs0, rd0, rc0, rs1, rd1, rc1, nruns, cur;
    int r_start, r_dir, r_left;
    unsigned long long clen;
    int cslot, cidx, ccount;
    bool crev;
    unsigned cphase;
    bool cwait;

    __device__ __forceinline__ void fill(int slot) {
        while (r_left == 0) {
            if (cur >= nruns) return;
            if (cur == 0) { r_start = rs0; r_dir = rd0; r_left = rc0; }
            else { r_start = rs1; r_dir = rd1; r_left = rc1; }
            ++cur;
        }
        const int cnt = r_left < kCH ? r_left : kCH;
        DMM_CHECK(slot >= 0 && slot < kNSlot && cnt >= 1 && cnt <= kCH);
        DMM_CHECK((r_dir > 0 ? r_start : r_start - cnt + 1) >= 0 &&
                  (r_dir > 0 ? r_start + cnt : r_start + 1) <= this->n);
        const unsigned sbase = ring + slot * slotB;
        const unsigned bar = mbar + 8 * slot;
        // every run is staged in ascending node order; a backward run is read
        // back to front (the rev bit)
        const unsigned long long rev = r_dir < 0 ? 0x80ull : 0ull;
        clen = (clen & ~(0xffull << (8 * slot))) | (((unsigned long long)cnt | rev) << (8 * slot));
        const bool box = VERT && this->vtma;   // V: one 2-D tensor box of kCH node rows
        if (this->lane == 0) mbar_expect_tx_s(bar, (unsigned)(2 * (box ? kCH : cnt) * SREC));
        __syncwarp();
        fence_proxy_async();
        __syncwarp();
        if constexpr (!VERT) {   // H: the A and B runs are contiguous -> two bulk copies (four across a segment edge)
            const int first = r_dir > 0 ? r_start : r_start - cnt + 1;
            const int n1 = this->run1(first, cnt, !FIRST);
            const int ln = this->lane;
            if (ln < 2 || (ln < 4 && n1 < cnt)) {
                const int c = (ln & 1) ? this->cB : this->cA;
                const int p = ln < 2 ? first : first + n1;
                const int nn = ln < 2 ? n1 : cnt - n1;
                tma_load_s(sbase + (ln & 1) * kOffB + (ln < 2 ? 0 : n1 * SREC),
                           this->src + this->srcq(c, p) * SREC, nn * SREC, bar);
            }
        } else {
            const int first = r_dir > 0 ? r_start : r_start - cnt + 1;
            if (box) {
                // rows first .. first + kCH - 1, bytes [cA*REC, cA*REC + 2*REC) of each
                // (rows past the run or the image are staged / zero-filled and unused)
                if (this->lane == 0)
                    tma_load_2d(sbase, this->P.tmap + 128 * (kCH == kRootCH ? 0 : 1), this->cA * (SREC / 8), first, bar);
            } else {
                const int k = this->lane & 15;
                if (k < cnt) {
                    const int p = first + k;
                    const size_t q = (size_t)this->qA(p);
                    if (this->hasB) {      // A and B adjacent in HBM
                        if (this->lane < 16) tma_load_s(sbase + k * kStride, this->src + q * SREC, 2 * SREC, bar);
                    } else {
                        tma_load_s(sbase + k * kStride + (this->lane < 16 ? 0 : SREC), this->src + q * SREC, SREC,
                                   bar);
                    }
                }
            }
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
    __device__ __forceinline__ void pop(unsigned (&v)[LPL], int& ba, int& bb) {
        if (cwait) chunk_wait();
        const unsigned ra = ring + cslot * slotB + (crev ? ccount - 1 - cidx : cidx) * kStride;
        this->dec(ra, ra + kOffB, v, ba, bb);
        if (++cidx == ccount) chunk_release();
    }
    // passes, as Task::run_pass in hm.cu.  Inside a chunk phi is left
    // unnormalised (min drifts up by <= span per step; pair_range_ok bounds
    // kChunkMax steps of drift); it is normalised at the chunk end and before
    // a spine store.
    template <int DIR>
    __device__ __forceinline__ void run_pass(int first, int nsteps, MP<LPL>& phi) {
        if (nsteps < 1) return;
        constexpr bool REV = DIR < 0;      // runs are staged in ascending node order
        const int len0 = nsteps + 1;
        int kk = DIR > 0 ? (31 - __clz(len0)) - 1 : 31 - __clz(len0 - 1);
        int target = DIR > 0 ? (len0 >> kk) : (((len0 - 1) >> kk) + 1);
        unsigned G = 0u;      // min of the current phi.m (packed)
        int gA = 0, gB = 0;
        auto normalise = [&]() {
#pragma unroll
            for (int e = 0; e < LPL; ++e) phi.m[e] = __vsub2(phi.m[e], G);
            phi.a += gA; phi.b += gB;
            G = 0u; gA = 0; gB = 0;
        };
        auto step = [&](const unsigned (&v)[LPL], int ba, int bb) {
#pragma unroll
            for (int e = 0; e < LPL; ++e) phi.m[e] += v[e];     // both >= 0 per half: no carry
            phi.a += ba; phi.b += bb;
            G = dtrans2<LPL, PAD, WIN, false>(phi.m, this->dk, gA, gB);
        };
        auto spine = [&](int s) {
            if (s + 2 == target) {
                normalise();
                this->st_spine(DIR > 0, first + DIR * (s + 1), phi);
                --kk;
                target = kk < 0 ? INT_MAX : (DIR > 0 ? (len0 >> kk) : (((len0 - 1) >> kk) + 1));
            }
        };
        int s = 0;
#pragma unroll 1
        while (s < nsteps) {
            chunk_wait();
            const unsigned base = ring + cslot * slotB;
            if (ccount == kCH && target - 2 >= s + kCH) {   // full chunk, no spine node: branch free
                unsigned v[LPL]; int ba, bb;
                {
                    const unsigned ra = base + (REV ? kCH - 1 : 0) * kStride;
                    this->dec(ra, ra + kOffB, v, ba, bb);
                }
#pragma unroll
                for (int k = 0; k < kCH; ++k) {
                    unsigned vn[LPL]; int ban = 0, bbn = 0;
                    if (k + 1 < kCH) {
                        const unsigned ra = base + (REV ? kCH - 2 - k : k + 1) * kStride;
                        this->dec(ra, ra + kOffB, vn, ban, bbn);
                    }
                    step(v, ba, bb);
                    if (k + 1 < kCH) {
#pragma unroll
                        for (int e = 0; e < LPL; ++e) v[e] = vn[e];
                        ba = ban; bb = bbn;
                    }
                }
                s += kCH;
            } else {                     // partial chunk or spine node inside: per step, next decode ahead
                const int cnt = ccount;
                const int st = REV ? -kStride : kStride;
                unsigned ra = base + (REV ? cnt - 1 : 0) * kStride;
                unsigned v[LPL]; int ba, bb;
                this->dec(ra, ra + kOffB, v, ba, bb);
#pragma unroll 1
                for (int k = 0; k < cnt; ++k) {
                    unsigned vn[LPL]; int ban, bbn;
                    ra += st;
                    const unsigned rn = k + 1 < cnt ? ra : base;   // in-bounds dummy on the last step
                    this->dec(rn, rn + kOffB, vn, ban, bbn);
                    step(v, ba, bb);
                    spine(s + k);
#pragma unroll
                    for (int e = 0; e < LPL; ++e) v[e] = vn[e];
                    ba = ban; bb = bbn;
                }
                s += cnt;
            }
            normalise();
            chunk_release();
        }
    }
    // Handshake; the ring delivers F_j then F_i.  Writes fwd[i+1] = phi_ij, bwd[i] = phi_ji'.
    template <bool OPT = false>
    __device__ __forceinline__ void handshake(int i, MP<LPL>& pl, MP<LPL>& pr, int* opt = nullptr) {
        unsigned vi[LPL], vj[LPL];
        int bia, bib, bja, bjb;
        pop(vj, bja, bjb);
        pop(vi, bia, bib);
        handshake2<LPL, PAD, WIN, OPT>(vi, bia, bib, vj, bja, bjb, pl, pr, this->dk, opt);
        this->st_spine(true, i + 1, pl);
        this->st_spine(false, i, pr);
    }
};

template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
__global__ void __launch_bounds__(64) hm2_root_kernel(PassArgs a) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int KP = 32 * LPL;
    const RingShared<kRootCH, kRootNS> lay(KP, FIRST);
    Task<LPL, VERT, PAD, WIN, FIRST, kRootCH, kRootNS> h;
    h.init(a, lane);
    h.set_pair(blockIdx.x);
    h.ring_init(smem + warp * lay.total, lay);
    pdl_wait();          // the node records were written by the previous half-step
    const int n = h.n, i = n / 2 - 1, j = i + 1;
    MP<LPL> zero, phi;
    zero.zero(); phi.zero();
    if (warp == 0) {
        h.rs0 = 0; h.rd0 = 1; h.rc0 = i;
        h.rs1 = j; h.rd1 = -1; h.rc1 = 2;
        h.start(2);
        h.st_spine(true, 0, zero);
        h.template run_pass<1>(0, i, phi);
    } else {
        h.rs0 = n - 1; h.rd0 = -1; h.rc0 = n - 1 - j;
        h.start(1);
        h.st_spine(false, n - 1, zero);
        h.template run_pass<-1>(n - 1, n - 1 - j, phi);
        h.st_spine(false, j, phi);
    }
    __syncthreads();
    if (warp == 0) {
        MP<LPL> pr;
        h.ld_spine(false, j, pr);
        int opt[2];
        h.template handshake<true>(i, phi, pr, opt);
        // the pair's share of the dual bound: the two chain optima (see handshake2)
        if (lane == 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(&h.P.bounds[a.bound_slot]),
                      (unsigned long long)((long long)opt[0] + (h.hasB ? (long long)opt[1] : 0ll)));
    }
    pdl_trigger_late();
}

template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST, int NW>
__global__ void __launch_bounds__(NW * 32, kLevMinCTAs) hm2_level_kernel(PassArgs a, int lev, int ntasks) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int KP = 32 * LPL;
    const RingShared<kLevCH, kLevNS> lay(KP, FIRST);
    Task<LPL, VERT, PAD, WIN, FIRST, kLevCH, kLevNS> h;
    h.init(a, lane);
    h.ring_init(smem + warp * lay.total, lay);
    const int n = h.n;
    bool waited = false;
#pragma unroll 1
    for (int t = blockIdx.x * NW + warp; t < ntasks; t += gridDim.x * NW) {
        h.set_pair(t >> lev);
        const int s = t & ((1 << lev) - 1);
        int lo, hi;
        task_bounds(n, lev, s, lo, hi);
        DMM_CHECK(lo >= 0 && hi < n && hi - lo >= 1);
        const int ii = lo + (hi - lo + 1) / 2 - 1, j = ii + 1;
        MP<LPL> bnd, spn;
        if (!(s & 1)) {   // left piece: reuse fwd, recompute bwd
            h.rs0 = hi; h.rd0 = -1; h.rc0 = hi - j;
            h.rs1 = j; h.rd1 = -1; h.rc1 = 2;
            h.start(2);
            if (!waited) { pdl_wait(); waited = true; }
            h.ld_spine(false, hi, bnd);
            h.ld_spine(true, ii, spn);
            h.template run_pass<-1>(hi, hi - j, bnd);
            h.handshake(ii, spn, bnd);
        } else {          // right piece: reuse bwd, recompute fwd
            h.rs0 = lo; h.rd0 = 1; h.rc0 = ii - lo;
            h.rs1 = j; h.rd1 = -1; h.rc1 = 2;
            h.start(2);
            if (!waited) { pdl_wait(); waited = true; }
            h.ld_spine(true, lo, bnd);
            h.ld_spine(false, j, spn);
            h.template run_pass<1>(lo, ii - lo, bnd);
            h.handshake(ii, bnd, spn);
        }
    }
    if (!waited) { pdl_wait(); }
    pdl_trigger_late();
}

// ======================================================== last level kernel
// The level just above the leaves (l* - 1): pieces of <= 2 kCMax nodes, so a
// task's pass (<= kCMax steps) and its Handshake pair fit one staging area of
// kLastRows node pairs, filled by one mbarrier phase (H: one bulk copy per
// chain; V: one 16-row tensor box) -- no ring, no chunk bookkeeping, no
// nested spine targets: the only spine message the leaves need from this
// pass is the one into their own first split (the leaf reuses it, "keep"),
// stored at its node; the Handshake outputs go to fwd[i+1] / bwd[i] as in the
// generic level kernel.  Same results (the same Msg sequence).
constexpr int kLastRows = 16;
static_assert(kLastRows >= kCMax + 2, "a last-level task stages its pass + Handshake nodes");

template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST, int NW>
__global__ void __launch_bounds__(NW * 32, kLevMinCTAs) hm2_last_kernel(PassArgs a, int lev, int ntasks) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    using PS = Pass<LPL, VERT, PAD, WIN, FIRST>;
    constexpr int SREC = PS::SREC;
    constexpr int kStride = VERT ? 2 * SREC : SREC, kOffB = VERT ? SREC : kLastRows * SREC;
    constexpr int kBytes = align_up(2 * kLastRows * SREC + 8, 128);
    char* wsm = smem + warp * kBytes;
    const unsigned sbase = smem_addr(wsm);
    const unsigned bar = sbase + 2 * kLastRows * SREC;
    if (lane == 0) { mbar_init(reinterpret_cast<uint64_t*>(wsm + 2 * kLastRows * SREC), 1); fence_mbar_init(); }
    __syncwarp();
    unsigned phase = 0;
    PS h;
    h.init(a, lane);
    const int n = h.n;
    bool waited = false;
#pragma unroll 1
    for (int t = blockIdx.x * NW + warp; t < ntasks; t += gridDim.x * NW) {
        h.set_pair(t >> lev);
        const int s = t & ((1 << lev) - 1);
        int lo, hi;
        task_bounds(n, lev, s, lo, hi);
        DMM_CHECK(lo >= 0 && hi < n && hi - lo + 1 <= 2 * kCMax + 1);
        const int ii = lo + (hi - lo + 1) / 2 - 1, j = ii + 1;
        const bool left = !(s & 1);
        const int s0 = left ? ii : lo, s1 = left ? hi : j;     // staged nodes, ascending
        const int cnt = s1 - s0 + 1;
        const bool box = VERT && h.vtma;
        if (lane == 0) mbar_expect_tx_s(bar, (unsigned)(2 * (box ? kLastRows : cnt) * SREC));
        __syncwarp();
        fence_proxy_async();
        __syncwarp();
        if constexpr (!VERT) {
            const int n1 = h.run1(s0, cnt, !FIRST);
            if (lane < 2 || (lane < 4 && n1 < cnt)) {
                const int c = (lane & 1) ? h.cB : h.cA;
                const int p = lane < 2 ? s0 : s0 + n1;
                tma_load_s(sbase + (lane & 1) * kOffB + (lane < 2 ? 0 : n1 * SREC), h.src + h.srcq(c, p) * SREC,
                           (lane < 2 ? n1 : cnt - n1) * SREC, bar);
            }
        } else if (box) {
            if (lane == 0) tma_load_2d(sbase, h.P.tmap, h.cA * (SREC / 8), s0, bar);
        } else if (lane < cnt) {
            const size_t q = (size_t)h.qA(s0 + lane);
            if (h.hasB) tma_load_s(sbase + lane * kStride, h.src + q * SREC, 2 * SREC, bar);
            else tma_load_s(sbase + lane * kStride, h.src + q * SREC, SREC, bar);
        }
        if (!waited) { pdl_wait(); waited = true; }
        MP<LPL> bnd, spn;
        if (left) { h.ld_spine(false, hi, bnd); h.ld_spine(true, ii, spn); }
        else { h.ld_spine(true, lo, bnd); h.ld_spine(false, j, spn); }
        mbar_wait_s(bar, phase);
        __syncwarp();
        phase ^= 1u;
        auto slot = [&](int p) { return sbase + (p - s0) * kStride; };
        // the pass: left piece backward from hi into j, right piece forward from lo into i
        const int dir = left ? -1 : 1;
        const int p0 = left ? hi : lo, steps = left ? hi - j : ii - lo;
        // the leaf's first-split message: right child [j, hi] of a left piece needs
        // the one into its split + 1 from the right; left child [lo, ii] of a right
        // piece the one into its split from the left (only for children of >= 4 nodes)
        const int lr = hi - j + 1, ll = ii - lo + 1;
        const int tgt = left ? (lr >= 4 ? j + lr / 2 : -1) : (ll >= 4 ? lo + ll / 2 - 1 : -1);
        unsigned v[LPL];
        int ba, bb;
        if (steps > 0) h.dec(slot(p0), slot(p0) + kOffB, v, ba, bb);
#pragma unroll 1
        for (int k = 0; k < steps; ++k) {
            const int p = p0 + dir * k;
            unsigned vn[LPL];
            int ban = 0, bbn = 0;
            const int pn = k + 1 < steps ? p + dir : p;    // in-bounds dummy on the last step
            h.dec(slot(pn), slot(pn) + kOffB, vn, ban, bbn);
#pragma unroll
            for (int e = 0; e < LPL; ++e) bnd.m[e] += v[e];
            bnd.a += ba; bnd.b += bb;
            h.msg_(bnd.m, bnd.a, bnd.b);                      // message into p + dir
            if (p + dir == tgt) h.st_spine(!left, tgt, bnd);
#pragma unroll
            for (int e = 0; e < LPL; ++e) v[e] = vn[e];
            ba = ban; bb = bbn;
        }
        // Handshake over (ii, j)
        unsigned vi[LPL], vj[LPL];
        int bia, bib, bja, bjb;
        h.dec(slot(ii), slot(ii) + kOffB, vi, bia, bib);
        h.dec(slot(j), slot(j) + kOffB, vj, bja, bjb);
        MP<LPL>& pl = left ? spn : bnd;
        MP<LPL>& pr = left ? bnd : spn;
        handshake2<LPL, PAD, WIN>(vi, bia, bib, vj, bja, bjb, pl, pr, h.dk);
        h.st_spine(true, ii + 1, pl);
        h.st_spine(false, ii, pr);
        __syncwarp();     // the staging area is refilled by the next task
    }
    if (!waited) { pdl_wait(); }
    pdl_trigger_late();
}

// ============================================================== leaf kernel
struct LeafShared {     // per-warp shared memory (bytes)
    int F, D, O, stack, mbar, total;
    __host__ __device__ LeafShared(int KP, bool first) {
        const int srec = first ? KP : rec_bytes(KP);
        F = 0;                                     // kCMax source record pairs
        D = F + 2 * kCMax * srec;                  // kCMax D-row pairs (unused when FIRST)
        // output record pairs: in place over F (a node's F is dead once it is
        // emitted), except when FIRST (F = D rows, shorter than a record)
        O = first ? D : F;
        stack = first ? O + 2 * kCMax * rec_bytes(KP) : D + 2 * kCMax * KP;   // kDepth x (phi_ij, R) message pairs
        mbar = align_up(stack + kDepth * 2 * (4 * KP + 16), 8);
        total = align_up(mbar + 8, 128);
    }
};

// stack entry: packed words [KP] u32 | int a | int b | 8 B pad
template <int LPL>
__device__ __forceinline__ void st_mp_s(uint8_t* p, int lane, const MP<LPL>& v) {
    constexpr int KP = 32 * LPL;
    st_i32<LPL>(reinterpret_cast<int32_t*>(p) + lane * LPL, reinterpret_cast<const int(&)[LPL]>(v.m));
    if (lane == 0) *reinterpret_cast<int2*>(p + 4 * KP) = make_int2(v.a, v.b);
}
template <int LPL>
__device__ __forceinline__ void ld_mp_s(const uint8_t* p, int lane, MP<LPL>& v) {
    constexpr int KP = 32 * LPL;
    ld_i32<LPL>(reinterpret_cast<const int32_t*>(p) + lane * LPL, reinterpret_cast<int(&)[LPL]>(v.m));
    const int2 o = *reinterpret_cast<const int2*>(p + 4 * KP);
    v.a = o.x; v.b = o.y;
}

// Emit leaf `node` of both chains: lambda = L + F + R (R8); the record
// L + R + D*2^F goes to the shared-memory output slots oa / ob (bulk-stored
// per block).  nodebound: bound += min lambda (only when no root Handshake
// supplied the chain optima, lstar == 0); last V: lowest argmin as the label
// (R13, R14).
template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
__device__ __forceinline__ void leaf_emit(const Pass<LPL, VERT, PAD, WIN, FIRST>& h, unsigned dA, unsigned dB,
                                          unsigned oA, unsigned oB, int node, const MP<LPL>& Lb, const MP<LPL>& Rb,
                                          const unsigned (&F)[LPL], int bfa, int bfb, bool last, bool nodebound,
                                          long long& bsum) {
    const int lane = h.lane;
    unsigned Dv[LPL], o[LPL];
    if constexpr (FIRST) {      // the unaries are D*2^F themselves
#pragma unroll
        for (int e = 0; e < LPL; ++e) Dv[e] = F[e];
    } else {
        ld_u8_pair_s<LPL>(dA, dB, lane, h.fbits, Dv);
    }
    unsigned lr[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        lr[e] = Lb.m[e] + Rb.m[e];
        o[e] = lr[e] + Dv[e];
    }
    const int oa = Lb.a + Rb.a, ob = Lb.b + Rb.b;
    st_rec_pair_s<LPL, PAD>(oA, oB, lane, o, oa, ob, h.K);
    if (nodebound || (VERT && last)) {
        unsigned lam[LPL];
        unsigned l = kBigP;
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            lam[e] = lr[e] + F[e];
            if (!PAD || lane * LPL + e < h.K) l = __vmins2(l, lam[e]);
        }
        const int gA = __reduce_min_sync(kFull, lo16(l)), gB = __reduce_min_sync(kFull, hi16(l));
        if (nodebound) {
            bsum += (long long)gA + oa + bfa;
            if (h.hasB) bsum += (long long)gB + ob + bfb;
        }
        if (VERT && last) {
            int ka = INT_MAX, kb = INT_MAX;
#pragma unroll
            for (int e = LPL - 1; e >= 0; --e) {
                const bool ok = !PAD || lane * LPL + e < h.K;
                if (ok && lo16(lam[e]) == gA) ka = lane * LPL + e;
                if (ok && hi16(lam[e]) == gB) kb = lane * LPL + e;
            }
            ka = __reduce_min_sync(kFull, ka);
            kb = __reduce_min_sync(kFull, kb);
            if (lane == 0) {
                h.P.labels[h.qA(node)] = (uint8_t)ka;
                if (h.hasB) h.P.labels[h.qB(node)] = (uint8_t)kb;
            }
        }
    }
}

// One warp per (chain pair, leaf block [lo, hi]) at level lstar: stage the
// block's record pairs, D rows and boundary messages, then solve its
// sub-hierarchy on chip, depth first (as hm_leaf_kernel in hm.cu).
template <int LPL, bool VERT, bool PAD, int WIN, bool FIRST>
__global__ void __launch_bounds__(kNWL * 32, DMM_LEAF_MINB) hm2_leaf_kernel(PassArgs a, int lstar, int nblocks) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    using PS = Pass<LPL, VERT, PAD, WIN, FIRST>;
    constexpr int KP = PS::KP, SREC = PS::SREC;
    constexpr int kStrideF = VERT ? 2 * SREC : SREC, kOffF = VERT ? SREC : kCMax * SREC;
    constexpr int kStrideD = FIRST ? kStrideF : (VERT ? 2 * KP : KP);
    constexpr int kOffD = FIRST ? kOffF : (VERT ? KP : kCMax * KP);
    constexpr int SMP = 4 * KP + 16;
    constexpr int REC = PS::REC;
    constexpr int kStrideO = VERT ? 2 * REC : REC, kOffO = VERT ? REC : kCMax * REC;
    const LeafShared lay(KP, FIRST);
    char* wsm = smem + warp * lay.total;
    const unsigned wsa = smem_addr(wsm);
    const unsigned sF = wsa + lay.F;
    const unsigned sD = FIRST ? sF : wsa + lay.D;
    const unsigned sO = wsa + lay.O;
    uint8_t* stk = reinterpret_cast<uint8_t*>(wsm + lay.stack);
    const unsigned bar = wsa + lay.mbar;
    if (lane == 0) { mbar_init(reinterpret_cast<uint64_t*>(wsm + lay.mbar), 1); fence_mbar_init(); }
    __syncwarp();
    unsigned phase = 0;
    const bool last = a.last != 0;
    const int nbl = 1 << lstar;
    long long bsum = 0;
    PS h;
    h.init(a, lane);
    const int n = h.n;
    const bool nodebound = lstar == 0;   // else the root Handshake added the chain optima
    bool waited = false;
    if (lstar == 0) {       // no root before this kernel: its records come from the previous kernel
        pdl_wait();
        waited = true;
    }

#pragma unroll 1
    for (int b = blockIdx.x * kNWL + warp; b < nblocks; b += gridDim.x * kNWL) {
        h.set_pair(b >> lstar);
        int lo0, hi0;
        task_bounds(n, lstar, b & (nbl - 1), lo0, hi0);
        const int m = hi0 - lo0 + 1;
        DMM_CHECK(lo0 >= 0 && hi0 < n && m >= 1 && m <= kCMax);
        const bool box = VERT && h.vtma;          // V: two 2-D tensor boxes of kCMax rows (records, D)
        const unsigned bytes = box ? 2 * kCMax * (SREC + KP) : 2 * m * SREC + (FIRST ? 0 : 2 * m * KP);
        bulk_wait_read();    // the previous block's output bulk stores have read the staging slots
        __syncwarp();
        if (lane == 0) mbar_expect_tx_s(bar, bytes);
        __syncwarp();
        fence_proxy_async();
        __syncwarp();
        if constexpr (!VERT) {
            const size_t qa = (size_t)h.qA(lo0), qb = (size_t)h.qB(lo0);
            const int n1 = h.run1(lo0, m, !FIRST);
            if (lane < 2 || (lane >= 4 && lane < 6 && n1 < m)) {
                const int c = (lane & 1) ? h.cB : h.cA;
                const int p = lane < 2 ? lo0 : lo0 + n1;
                tma_load_s(sF + (lane & 1) * kOffF + (lane < 2 ? 0 : n1 * SREC), h.src + h.srcq(c, p) * SREC,
                           (lane < 2 ? n1 : m - n1) * SREC, bar);
            }
            if (!FIRST && lane == 2) tma_load_s(sD, h.P.D + qa * KP, m * KP, bar);
            if (!FIRST && lane == 3) tma_load_s(sD + kOffD, h.P.D + qb * KP, m * KP, bar);
        } else if (box) {
            if (lane == 0) tma_load_2d(sF, h.P.tmap + 256, h.cA * (SREC / 8), lo0, bar);
            if (lane == 1) tma_load_2d(sD, h.P.tmap + 384, h.cA * (KP / 8), lo0, bar);
        } else {
            const int k = lane & 15;
            if (k < m) {
                const size_t q = (size_t)h.qA(lo0 + k);
                if (h.hasB) {
                    if (lane < 16) tma_load_s(sF + k * kStrideF, h.src + q * SREC, 2 * SREC, bar);
                    else if (!FIRST) tma_load_s(sD + k * kStrideD, h.P.D + q * KP, 2 * KP, bar);
                } else {
                    const unsigned hb = lane < 16 ? 0u : 1u;
                    tma_load_s(sF + k * kStrideF + hb * SREC, h.src + q * SREC, SREC, bar);
                    if (!FIRST) tma_load_s(sD + k * kStrideD + hb * KP, h.P.D + q * KP, KP, bar);
                }
            }
        }
        if (!waited) { pdl_wait(); waited = true; }
        MP<LPL> L, R, Kp;
        // Fig.11 reuse for the block's first split: a left block keeps its left
        // boundary, so the message into its split node from the left is on the
        // fwd spine (stored by the pass that produced L); a right block finds the
        // one from the right on the bwd spine.  Only the other pass is computed.
        int keep = 0;
        if (lstar > 0) {
            h.ld_spine(true, lo0, L);
            h.ld_spine(false, hi0, R);
            if (m >= 4) {
                const int ib = m / 2 - 1;
                if (!(b & 1)) { h.ld_spine(true, lo0 + ib, Kp); keep = 1; }
                else { h.ld_spine(false, lo0 + ib + 1, Kp); keep = 2; }
            }
        } else {
            L.zero(); R.zero();
        }
        mbar_wait_s(bar, phase);
        __syncwarp();
        phase ^= 1u;
        auto fA = [&](int k) { return sF + k * kStrideF; };
        auto dA = [&](int k) { return sD + k * kStrideD; };
        auto emit = [&](int k, const MP<LPL>& Lb, const MP<LPL>& Rb, const unsigned (&F)[LPL], int ba, int bb) {
            const unsigned oa = sO + k * kStrideO;
            leaf_emit<LPL, VERT, PAD, WIN, FIRST>(h, dA(k), dA(k) + kOffD, oa, oa + kOffO, lo0 + k, Lb, Rb, F, ba, bb,
                                                  last, nodebound, bsum);
        };
        // pieces of <= 3 nodes: straight-line code (R5 with the splits unrolled)
        auto small = [&](int lo, int hi, const MP<LPL>& L, const MP<LPL>& R) {
            unsigned F0[LPL]; int b0a, b0b;
            h.dec(fA(lo), fA(lo) + kOffF, F0, b0a, b0b);
            if (lo == hi) {
                emit(lo, L, R, F0, b0a, b0b);
                return;
            }
            unsigned F1[LPL]; int b1a, b1b;
            h.dec(fA(lo + 1), fA(lo + 1) + kOffF, F1, b1a, b1b);
            MP<LPL> pl = L, pr = R;
            unsigned F2[LPL]; int b2a = 0, b2b = 0;
            if (hi == lo + 2) {                 // [lo, lo+2]: i = lo, j = lo+1; one backward step
                h.dec(fA(lo + 2), fA(lo + 2) + kOffF, F2, b2a, b2b);
#pragma unroll
                for (int e = 0; e < LPL; ++e) pr.m[e] += F2[e];
                pr.a += b2a; pr.b += b2b;
                h.msg_(pr.m, pr.a, pr.b);
            }
            handshake2<LPL, PAD, WIN>(F0, b0a, b0b, F1, b1a, b1b, pl, pr, h.dk);
            emit(lo, L, pr, F0, b0a, b0b);      // A = [lo, lo] (L, phi_ji')
            if (hi == lo + 1) {
                emit(lo + 1, pl, R, F1, b1a, b1b);
            } else {                            // B = [lo+1, lo+2] (phi_ij, R): i = lo+1, j = lo+2
                MP<LPL> ql = pl, qr = R;
                handshake2<LPL, PAD, WIN>(F1, b1a, b1b, F2, b2a, b2b, ql, qr, h.dk);
                emit(lo + 1, pl, qr, F1, b1a, b1b);
                emit(lo + 2, ql, R, F2, b2a, b2b);
            }
        };
        int lo = 0, hi = m - 1, sp = 0;
        unsigned stkJ = 0, stkH = 0;
#pragma unroll 1
        while (true) {
            if (hi - lo < 3) {
                small(lo, hi, L, R);
                if (sp == 0) break;
                --sp;
                lo = (int)((stkJ >> (kFB * sp)) & ((1u << kFB) - 1));
                hi = (int)((stkH >> (kFB * sp)) & ((1u << kFB) - 1));
                __syncwarp();
                ld_mp_s<LPL>(stk + (2 * sp) * SMP, lane, L);
                ld_mp_s<LPL>(stk + (2 * sp + 1) * SMP, lane, R);
                continue;
            }
            const int len = hi - lo + 1, i = lo + len / 2 - 1, j = i + 1;
            MP<LPL> pl = L, pr = R;
            // the two passes interleaved (independent chains -> ILP), left
            // unnormalised until the Handshake (<= 5 steps of drift)
            const int nf = i - lo, nb = hi - j;     // nb == nf or nf + 1
            unsigned Gl = 0u, Gr = 0u;
            int gla = 0, glb = 0, gra = 0, grb = 0;
            auto stepL = [&](int k) {
                unsigned F[LPL]; int ba, bb;
                h.dec(fA(k), fA(k) + kOffF, F, ba, bb);
#pragma unroll
                for (int e = 0; e < LPL; ++e) pl.m[e] += F[e];
                pl.a += ba; pl.b += bb;
                Gl = dtrans2<LPL, PAD, WIN, false>(pl.m, h.dk, gla, glb);
            };
            auto stepR = [&](int k) {
                unsigned F[LPL]; int ba, bb;
                h.dec(fA(k), fA(k) + kOffF, F, ba, bb);
#pragma unroll
                for (int e = 0; e < LPL; ++e) pr.m[e] += F[e];
                pr.a += ba; pr.b += bb;
                Gr = dtrans2<LPL, PAD, WIN, false>(pr.m, h.dk, gra, grb);
            };
            const int kp = keep;
            keep = 0;
            if (kp == 1) {                  // phi into i from the left: fwd spine
                pl = Kp;
#pragma unroll 1
                for (int s = 0; s < nb; ++s) stepR(hi - s);
            } else if (kp == 2) {           // phi into j from the right: bwd spine
                pr = Kp;
#pragma unroll 1
                for (int s = 0; s < nf; ++s) stepL(lo + s);
            } else {
#pragma unroll 1
                for (int s = 0; s < nf; ++s) { stepL(lo + s); stepR(hi - s); }
                if (nb > nf) stepR(hi - nf);
            }
#pragma unroll
            for (int e = 0; e < LPL; ++e) { pl.m[e] = __vsub2(pl.m[e], Gl); pr.m[e] = __vsub2(pr.m[e], Gr); }
            pl.a += gla; pl.b += glb; pr.a += gra; pr.b += grb;
            unsigned Fi[LPL], Fj[LPL];
            int bia, bib, bja, bjb;
            h.dec(fA(i), fA(i) + kOffF, Fi, bia, bib);
            h.dec(fA(j), fA(j) + kOffF, Fj, bja, bjb);
            handshake2<LPL, PAD, WIN>(Fi, bia, bib, Fj, bja, bjb, pl, pr, h.dk);
            // children A = (lo, i, L, phi_ji' = pr), B = (j, hi, phi_ij = pl, R), both >= 2
            // nodes: push B, continue with A
            DMM_CHECK(sp < kDepth);
            stkJ = (stkJ & ~(((1u << kFB) - 1) << (kFB * sp))) | ((unsigned)j << (kFB * sp));
            stkH = (stkH & ~(((1u << kFB) - 1) << (kFB * sp))) | ((unsigned)hi << (kFB * sp));
            __syncwarp();
            st_mp_s<LPL>(stk + (2 * sp) * SMP, lane, pl);
            st_mp_s<LPL>(stk + (2 * sp + 1) * SMP, lane, R);
            ++sp;
            hi = i;
            R = pr;
        }
        // the block's output records: bulk stores from the staging slots
        __syncwarp();
        fence_proxy_async();
        __syncwarp();
        if constexpr (!VERT) {
            const int n1 = h.run1(lo0, m, true);
            if ((lane < 2 || (lane < 4 && n1 < m)) && ((lane & 1) == 0 || h.hasB)) {
                const int c = (lane & 1) ? h.cB : h.cA;
                const int p = lane < 2 ? lo0 : lo0 + n1;
                tma_store_s(h.dst + h.rq(c, p) * REC, sO + (lane & 1) * kOffO + (lane < 2 ? 0 : n1 * REC),
                            (lane < 2 ? n1 : m - n1) * REC);
            }
        } else {
            if (lane < m) tma_store_s(h.dst + (size_t)h.qA(lo0 + lane) * REC, sO + lane * kStrideO,
                                      (h.hasB ? 2 : 1) * REC);
        }
        bulk_commit();
    }
    bulk_wait_all();
    if (!waited) pdl_wait();
    if (lane == 0 && bsum != 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&h.P.bounds[a.bound_slot]), (unsigned long long)bsum);
    pdl_trigger_late();
}

// ================================================================ launchers
static int leaf_level(int n) {
    int l = 0;
    while (((n + (1 << l) - 1) >> l) > kCMax) ++l;
    return l;
}

// Launch with programmatic stream serialisation (see pdl_wait /
// pdl_trigger_late), every label width.
template <typename... KArgs, typename... Args>
static void launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// Per-instantiation launch constants (SM count, occupancy, smem opt-in),
// queried once per device: host API calls between the ~8 launches of a
// half-step would otherwise starve the GPU.
struct LaunchCache {
    int dev = -1, sms = 148, lev_cap = 148, leaf_cap = 148, last_cap = 148;
};
#ifndef DMM_USE_LAST
#define DMM_USE_LAST 1
#endif
constexpr bool kUseLast = DMM_USE_LAST;

template <int LPL, bool PAD, int WIN, bool FIRST, bool VERT>
static void launch_cfg(const PassArgs& a, int nframes, cudaStream_t s) {
    constexpr int KP = 32 * LPL;
    constexpr int kNWG = nwg<LPL>();
    const int chains = VERT ? a.L.W : a.L.H;
    const int units = (chains + 1) / 2;      // chain pairs
    const int n = VERT ? a.L.H : a.L.W;
    const int lstar = leaf_level(n);
    const int rr = RingShared<kRootCH, kRootNS>(KP, FIRST).total;
    const int rs = RingShared<kLevCH, kLevNS>(KP, FIRST).total;
    const int smem = kNWL * LeafShared(KP, FIRST).total;
    auto rk = hm2_root_kernel<LPL, VERT, PAD, WIN, FIRST>;
    auto lk = hm2_level_kernel<LPL, VERT, PAD, WIN, FIRST, kNWG>;
    auto kern = hm2_leaf_kernel<LPL, VERT, PAD, WIN, FIRST>;
    auto lastk = hm2_last_kernel<LPL, VERT, PAD, WIN, FIRST, kNWG>;
    const int rl = align_up(2 * kLastRows * (FIRST ? KP : rec_bytes(KP)) + 8, 128);
    static LaunchCache lc;
    int dev = 0;
    cudaGetDevice(&dev);
    if (lc.dev != dev) {
        cudaDeviceGetAttribute(&lc.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * rr);
        cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, kNWG * rs);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(lastk, cudaFuncAttributeMaxDynamicSharedMemorySize, kNWG * rl);
        int per_sm_last = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_last, lastk, kNWG * 32, kNWG * rl);
        lc.last_cap = lc.sms * (per_sm_last > 0 ? per_sm_last : 1);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lk, kNWG * 32, kNWG * rs);
        lc.lev_cap = lc.sms * (per_sm > 0 ? per_sm : 1);
        per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNWL * 32, smem);
        lc.leaf_cap = lc.sms * (per_sm > 0 ? per_sm : 1);
        lc.dev = dev;
    }
    if (lstar > 0) {
        launch_pdl(true, rk, dim3(units, nframes), 64, 2 * rr, s, a);
        for (int lev = 1; lev < lstar; ++lev) {
            const int ntasks = units << lev;
            if (lev == lstar - 1 && kUseLast) {      // pieces of <= 2 kCMax nodes: the ring-free kernel
                int grid = (ntasks + kNWG - 1) / kNWG;
                if (grid > lc.last_cap) grid = lc.last_cap;
                launch_pdl(true, lastk, dim3(grid, nframes), kNWG * 32, kNWG * rl, s, a, lev, ntasks);
                continue;
            }
            int grid = (ntasks + kNWG - 1) / kNWG;
            if (grid > lc.lev_cap) grid = lc.lev_cap;
            launch_pdl(true, lk, dim3(grid, nframes), kNWG * 32, kNWG * rs, s, a, lev, ntasks);
        }
    }
    const int nblocks = units << lstar;
    int grid = (nblocks + kNWL - 1) / kNWL;
    if (grid > lc.leaf_cap) grid = lc.leaf_cap;
    launch_pdl(true, kern, dim3(grid, nframes), kNWL * 32, smem, s, a, lstar, nblocks);
}

template <int LPL, bool PAD, int WIN>
static void launch_dir(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    if (vertical) launch_cfg<LPL, PAD, WIN, false, true>(a, nframes, s);
    else if (a.first) launch_cfg<LPL, PAD, WIN, true, false>(a, nframes, s);
    else launch_cfg<LPL, PAD, WIN, false, false>(a, nframes, s);
}

template <int LPL, bool PAD>
void launch_win(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    if (a.T > LPL + 1) launch_dir<LPL, PAD, 0>(a, vertical, nframes, s);
    else if constexpr (LPL >= 4) {
        if (a.T == 4) launch_dir<LPL, PAD, 4>(a, vertical, nframes, s);
        else launch_dir<LPL, PAD, -1>(a, vertical, nframes, s);
    } else {
        launch_dir<LPL, PAD, -1>(a, vertical, nframes, s);
    }
}

}  // namespace p2
}  // namespace dmm
