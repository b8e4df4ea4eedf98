"""The C++ drop-in layer (include/spten/gpu.hpp): run the C++ parity suite
(tests/cpp/test_dropin.cpp) that compares spten::gpu::* with the real
reference's spten::seq::* through the reference's own types and predicates."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin.bin")
LIB = os.path.join(ROOT, "paper_1902_03317_b200", "libspten_gpu.so")


def test_dropin_library_links_the_c_abi():
    """CPU-side: the drop-in .so exists and depends on the C-ABI library."""
    if not os.path.exists(LIB):
        pytest.skip("drop-in layer not built (needs the reference headers)")
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    for sym in ("spten::gpu::mttkrp", "spten::gpu::tew_eq", "spten::gpu::tew", "spten::gpu::ts",
                "spten::gpu::ttv", "spten::gpu::ttm", "spten::gpu::sort_lexicographic",
                "spten::gpu::coalesce", "spten::gpu::build_fiber_index", "spten::gpu::read_tns"):
        assert sym in out, sym
    und = subprocess.run(["nm", "-D", "--undefined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    assert "spt_mttkrp_f32" in und and "spt_tew_f32" in und


@pytest.mark.gpu
def test_cpp_dropin_parity_suite():
    if not os.path.exists(BIN):
        pytest.skip("C++ parity binary not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
