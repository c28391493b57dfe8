"""Seeded fuzz of the drop-in path against the oracle (tools/fuzz_parity.py): random orders 2-5,
extents from 1, ranks above and below the extents, p, q from 0, both stabilizers and sketch
distributions, mode subsets including the empty one. Every case must meet the bars
(fp64: compressed tensor, relerr and factors within 1e-8 relative, equal iterations; fp32: fit within 1e-4) or raise the
same error message on both sides."""
import os
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


@pytest.mark.parametrize("seed,dtype", [(2024, "f64"), (7, "f64"), (11, "f32")])
def test_fuzz_compress_and_decompose(rcp, oracle, seed, dtype):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_parity
    import numpy as np
    flagged = []
    bad = fuzz_parity.run(150, seed, out=lambda *a: flagged.append(" ".join(str(x) for x in a)),
                          dtype=np.float32 if dtype == "f32" else np.float64)
    assert bad == 0, "\n".join(flagged)
