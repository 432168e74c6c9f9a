/*
 * dmm_oracle.h -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 1601.06274 (Shekhovtsov, Reinbacher, Graber, Pock, CVWW 2016):
 * census cost volume + Dual MM (Algorithm 2) with hierarchical minorants
 * (Handshake, Algorithm 5).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1601_06274_b200/csrc), and neither side includes the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (+ section / equation).
 * Readings of silent or garbled passages are listed in DESIGN.md "Readings".
 *
 * All cost arithmetic is exact integer (int64).  Energies / bounds are in
 * units of 2^-Fbits (fixed point), reading R9.
 * Layouts: images / codes / labels are row-major [H][W]; cost volumes and
 * duals are label-contiguous [H][W][K] (dense, no padding).
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (brute force, closed forms, paper-printed values); none is "parity unpinned".
 */
#ifndef DMM_ORACLE_H
#define DMM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Census transform (Sec. 3.1; reading R17): bit b, in raster order over
 * the (2r+1)^2 window offsets skipping the centre, is [I(nbr) < I(centre)];
 * neighbours outside the image replicate the border.  r in {1,2}.
 * Returns 0, or 1 on bad arguments. */
int oracle_census(const uint8_t* img, int W, int H, int r, uint32_t* codes);

/* Hamming cost volume ("f_i(x_i) = D_i(u(x_i))"):
 * D[y][x][k] = popcount(cl[y][x] ^ cr[y][x-d_k]), d_k = d_min + k,
 * or oob when x-d_k is outside [0,W).  Returns 0 / 1 (bad args). */
int oracle_cost_volume(const uint32_t* cl, const uint32_t* cr, int W, int H,
                       int d_min, int K, int oob, uint8_t* D);

/* Optimistic decoupled flow costs (Eq. "flow decoupled costs", P:163-170;
 * Sec. 3.2 P:442-447 "decoupled into two independent stereo-like problems"),
 * by plain enumeration of the 2-D label window: with displacements
 * u1(a) = u1_min + a (a < K1, horizontal) and u2(b) = u2_min + b (b < K2,
 * vertical), D(a,b) = popcount(c1[y][x] ^ c2[y+u2(b)][x+u1(a)]) or oob when
 * the displaced pixel leaves the image (readings R22, R23), and
 *   f1[y][x][a] = min_b D(a,b),   f2[y][x][b] = min_a D(a,b).
 * f1 is [H][W][K1], f2 is [H][W][K2].  Returns 0 / 1 (bad args). */
int oracle_flow_costs(const uint32_t* c1, const uint32_t* c2, int W, int H, int u1_min, int K1,
                      int u2_min, int K2, int oob, uint8_t* f1, uint8_t* f2);

/* Message passing, definition (P:663-667 Eq. msg-pass; Msg in Alg.5):
 * out(b) = min_a a(a) + ws*min(|a-b|, T), by direct O(K^2) enumeration. */
void oracle_msg_direct(const int64_t* a, int K, int64_t ws, int T, int64_t* out);

/* Same message by the O(K) lower-envelope distance transform for the
 * truncated-linear term (forward pass, backward pass, min with min(a)+ws*T). */
void oracle_msg(const int64_t* a, int K, int64_t ws, int T, int64_t* out);

/* Min-marginals of a chain (Def. P:631-636, Eq. P:646-649):
 * m_i = phi_{i-1,i} + F_i + phi_{i+1,i}.  F, m are [n][K]. */
void oracle_min_marginals(const int64_t* F, int n, int K, int64_t ws, int T, int64_t* m);

/* Chain optimum min_x sum_i F_i(x_i) + sum ws*min(|x_i-x_{i+1}|,T) by plain
 * Viterbi (never calls the minorant code).  x_opt (nullable) receives the
 * lexicographically smallest optimal labelling. */
int64_t oracle_chain_min(const int64_t* F, int n, int K, int64_t ws, int T, int32_t* x_opt);

/* Hierarchical minorant of one chain (Handshake Alg.5 P:811-830,
 * schedule Fig.11), reading R5/R7/R8/R9/R10 of DESIGN.md.
 * lam is [n][K]. */
void oracle_hm(const int64_t* F, int n, int K, int64_t ws, int T, int64_t* lam);

/* Dual MM (Algorithm 2) on the 4-connected grid with all unaries in
 * the horizontal subproblem f and vertical pairwise in g (reading R3), initial
 * g_ = 0 (R4), `iters` full iterations (H half-step then V half-step, R5).
 *   D       u8 [H][W][K] cost volume (unscaled).
 *   pairwise f_ij = w * min(|a-b|, T) (w = w_h or w_v), all scaled by 2^Fbits.
 *   fdual, gdual (nullable): int64 [H][W][K], the minorants f_, g_ after the
 *     last H resp. V half-step of the last iteration.
 *   labels (nullable): int32 [H][W], lowest-index argmin of the last V
 *     minorant (R13, R14).
 *   bound_hist (nullable): int64 [2*iters], b_{2t} after H, b_{2t+1} after V.
 *   energy (nullable): E(labels) * 2^Fbits.
 * nthreads <= 1 runs single-threaded.  Returns 0, or 1 on bad arguments. */
int oracle_dmm(const uint8_t* D, int W, int H, int K, int w_h, int w_v, int T,
               int Fbits, int iters, int64_t* fdual, int64_t* gdual,
               int32_t* labels, int64_t* bound_hist, int64_t* energy, int nthreads);

/* Primal energy Eq.3 of a labelling, unscaled:
 * sum_i D_i(x_i) + w_h sum_h min(|x_i-x_j|,T) + w_v sum_v min(|x_i-x_j|,T). */
int64_t oracle_energy(const uint8_t* D, const int32_t* labels, int W, int H, int K,
                      int w_h, int w_v, int T);

/* ---- NEXT-3: general penalty and edge weights (Fig.2; Eq.
 * regularizer-form P:134-136; r-decompose P:364-375), readings R29-R31.
 * R(d) = min(e1*min(d, delta) + e2*max(d - delta, 0), c)   (integers, units 2^-F:
 *   slope e1 = eps*2^F up to delta, slope e2 = 2^F beyond, truncated at c = C*2^F),
 * edge (i,j) of direction w (w_h / w_v) with quantised weight om in [1, 16]:
 *   V_ij(d) = floor(w * om * R(|d|) / 16)   (om = 16: constant weights).
 * With e1 = e2 = 2^F, c = T*2^F and om = 16 this is w*min(|d|,T)*2^F. */
typedef struct { int32_t e1, e2, delta, c; } oracle_pen;

/* Edge-aware weights (SPEC S:99 formula, quantised, reading R30):
 * om(g) = clamp(round(16 exp(-5 g / 255)), 1, 16), g = |I_i - I_j| (u8).
 * om_h[y][x]: edge (y,x)-(y,x+1); om_v[y][x]: edge (y,x)-(y+1,x); the last
 * column / row entries are 16 (unused). */
void oracle_edge_weights(const uint8_t* img, int W, int H, uint8_t* om_h, uint8_t* om_v);

/* Dual MM (Algorithm 2) with the general pairwise term above: the same
 * algorithm as oracle_dmm with every Msg = min_a a(a) + V_ij(|a-b|) by
 * direct enumeration over the edge's own V (Alg.5 literal, three Msg per
 * Handshake).  om_h / om_v nullable (= all 16).  Outputs as oracle_dmm;
 * energy = D*2^F + sum V (already scaled).  Returns 0 / 1 (bad args). */
int oracle_dmm_general(const uint8_t* D, int W, int H, int K, int w_h, int w_v, oracle_pen pen,
                       const uint8_t* om_h, const uint8_t* om_v, int Fbits, int iters, int64_t* fdual,
                       int64_t* gdual, int32_t* labels, int64_t* bound_hist, int64_t* energy, int nthreads);
/* Energy of a labelling under the general model (scaled by 2^F). */
int64_t oracle_energy_general(const uint8_t* D, const int32_t* labels, int W, int H, int K, int w_h, int w_v,
                              oracle_pen pen, const uint8_t* om_h, const uint8_t* om_v, int Fbits);
/* Hierarchical minorant of one chain under the general model: om[n-1] edge
 * weights (nullable = 16), w the direction weight. */
void oracle_hm_general(const int64_t* F, int n, int K, int w, oracle_pen pen, const uint8_t* om, int64_t* lam);

/* ---- NEXT-4 minorant variants (readings R32, R33).
 * Iterative minorant, Alg.4: max_pass passes alternating
 * direction (first: node 0 -> n-1), lambda_i += floor(m_i / 2^gshift) with the
 * dynamic min-marginal m_i of f - lambda, the last pass with gamma = 1
 * (the paper's run: max_pass = 3, gamma = 0.25).
 * Naive minorant: lambda = floor(min-marginals of f / n). */
void oracle_iter_minorant(const int64_t* F, int n, int K, int w, oracle_pen pen, const uint8_t* om, int max_pass,
                          int gshift, int64_t* lam);
void oracle_naive_minorant(const int64_t* F, int n, int K, int w, oracle_pen pen, const uint8_t* om, int64_t* lam);
/* Dual MM with minorant 0 = hierarchical (= oracle_dmm_general), 1 =
 * iterative (max_pass, gshift), 2 = naive. */
int oracle_dmm_minorant(const uint8_t* D, int W, int H, int K, int w_h, int w_v, oracle_pen pen,
                        const uint8_t* om_h, const uint8_t* om_v, int Fbits, int iters, int minorant, int max_pass,
                        int gshift, int64_t* fdual, int64_t* gdual, int32_t* labels, int64_t* bound_hist,
                        int64_t* energy, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
