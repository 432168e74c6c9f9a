"""Writes tests/golden/hm_chains.json: hierarchical-minorant values (HM, reading
R5/R7/R9 of DESIGN.md, Handshake Alg.5) on odd-length and
deeper chains (n = 7, 13, 25) at F = 0 and F = 4.

Calls only oracle/ (it never touches the CUDA path).  The values are regression
goldens for the oracle and for the GPU (tests/test_gpu_parity.py); they are
pinned independently of the oracle by tests/test_oracle_chain.py:
  * brute force (valid, exact, maximal minorant) on the n = 7 chains;
  * the recursive optimum split (a consequence of floor halving, R9, and the
    floor(len/2) split, R7): every piece of the recursion with optimum O gives
    its left part ceil(O/2) and its right part floor(O/2);
  * the first Handshake of the n = 7, F = 0 chain worked by hand in the JSON's
    "_hand_check" entry against Alg.5's four lines.

Run:  python tests/golden/make_hm_chains.py
"""
import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


# Worked by hand (not by this script's oracle calls); the test checks the
# oracle's lambda for chains[0] is consistent with it (top-level optimum split).
HAND_CHECK = {
    "chain": "chains[0] (n = 7, F = 0, K = 5, w = 3, T = 2); top-level split i = 2, j = 3 "
             "(R7: left part floor(7/2) = 3 nodes)",
    "how": "Worked by hand with the O(K^2) definition of Msg (Eq. msg-pass P:663-667, f_ij = 3 min(|a-b|, 2)) "
           "and the four lines of Alg.5 (P:811-830, readings R9/R10). E.g. Msg(D_0) = [8, 6, 9, 7, 10]; "
           "+ D_1 = [28, 23, 20, 8, 28]; Msg -> [14, 14, 11, 8, 11].",
    "phi_into_i_from_left": [14, 14, 11, 8, 11],
    "phi_into_j_from_right": [18, 18, 15, 17, 20],
    "alg5_line1_phi_ji": [25, 28, 27, 25, 28],
    "alg5_line2_m_i": [59, 58, 45, 35, 61],
    "alg5_line3_floor_half_m_i_minus_2phi_ji": [4, 1, -5, -8, 2],
    "alg5_line3_phi_ij": [-2, -2, -5, -8, -5],
    "alg5_line4_phi_ji_bounced": [2, 2, 5, 8, 5],
    "left_part_optimum": 18, "right_part_optimum": 17, "chain_optimum": 35,
    "note": "min m_i = 35 = chain optimum; the left part keeps ceil(35/2) = 18, the right part "
            "floor(35/2) = 17 (floor halving, R9)",
}


def main():
    rng = np.random.default_rng(20260)
    out = {"_source": "tests/golden/make_hm_chains.py (calls only oracle/: oracle.hm, oracle.chain_min)",
           "K": 5, "w": 3, "T": 2, "chains": []}
    for n in (7, 13, 25):
        D = rng.integers(0, 25, size=(n, 5))          # census-range unaries (5x5: 0..24)
        for F in (0, 4):
            ws = 3 << F
            lam = oracle.hm(D << F, ws, 2)
            opt = oracle.chain_min(D << F, ws, 2)[0]
            out["chains"].append({"n": n, "F": F, "D": D.tolist(), "lam": lam.tolist(), "opt": int(opt)})
    out["_hand_check"] = HAND_CHECK
    text = json.dumps(out, indent=1)
    # one matrix row per line
    text = re.sub(r"\[\s+([-\d,\s]+?)\s+\]", lambda m: "[" + " ".join(m.group(1).split()) + "]", text)
    with open(os.path.join(HERE, "hm_chains.json"), "w") as f:
        f.write(text + "\n")


if __name__ == "__main__":
    main()
