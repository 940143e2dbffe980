"""FAQ 4 workload switch (SPEC.md:284-287 select_path) through
the C ABI — host logic only, no GPU needed.  Golden cases are SPEC.md's
examples."""
import pytest

import paper_2403_08845_b200 as ba
from paper_2403_08845_b200 import _build


@pytest.fixture(scope="module", autouse=True)
def _lib():
    _build.build()


def _p(b, mc, md=0):
    return ba.make_problem(b, 32, 32, 128, mc, md, 0)


def test_spec_examples():
    # SPEC.md:290 mode=auto, threshold=4096, b=1, m_c=128 -> naive
    assert ba.select_path(_p(1, 128), "auto", 4096) == "naive"
    # SPEC.md:291 mode=auto, threshold=4096, b=16, m_c=8192 -> bifurcated
    assert ba.select_path(_p(16, 8192), "auto", 4096) == "bifurcated"
    # SPEC.md:292 mode=always_bifurcated, any workload -> bifurcated
    assert ba.select_path(_p(1, 1), "always_bifurcated") == "bifurcated"
    assert ba.select_path(_p(64, 65536), "always_naive") == "naive"


def test_threshold_is_strict_on_b_times_mc():
    assert ba.select_path(_p(4, 1024), "auto", 4096) == "naive"        # 4096 is not > 4096
    assert ba.select_path(_p(4, 1025), "auto", 4096) == "bifurcated"
    assert ba.select_path(_p(1, 4097), "auto", 4096) == "bifurcated"   # md does not enter
    assert ba.select_path(_p(1, 4096, md=10**5), "auto", 4096) == "naive"


def test_default_threshold_and_bad_inputs():
    assert ba.select_path(_p(32, 8192), "auto") == "bifurcated"       # C2b
    assert ba.select_path(_p(1, 64), "auto") == "naive"
    with pytest.raises(ba.BifAttnError):
        ba.select_path(ba.make_problem(1, 3, 2, 128, 10, 0, 0), "auto")  # h % g != 0
