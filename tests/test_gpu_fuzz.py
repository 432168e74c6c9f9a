"""A fixed, seeded slice of the randomised GPU-vs-oracle parity run
(tests/fuzz_parity.py): 400 random configurations over every path -- the
classic pair / int32 kernels, the general penalty with edge weights, the
iterative minorant, flow costs + layers + flow refinement, stereo refinement,
ROWCOL bands in lockstep -- each compared exactly as the parity tests do."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_fuzz_slice():
    pytest.importorskip("torch")
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import fuzz_parity
    n, counts, _ = fuzz_parity.run(budget=600.0, seed=2024, scale=1, max_cases=400, verbose=False)
    assert n == 400 and len(counts) == 5, counts
