"""The C++ mirror API (include/knn_b200/bruteforce.hpp) and the reference-side
drop-in (integration/knn_bf_knn_b200.cpp linked into the reference build in
place of src/bruteforce.cpp, driving the reference's own callers)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM_TEST = os.path.join(ROOT, "tests", "cpp", "test_bruteforce_b200")
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


def _build_shim_test():
    if not os.path.exists(SHIM_TEST):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_mirror_contract_errors_host_only():
    """test_bruteforce.cpp:92-102 contract errors: validated on the host, no GPU needed."""
    _build_shim_test()
    r = subprocess.run([SHIM_TEST, "--no-gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_mirror_reference_unit_cases():
    _build_shim_test()
    r = subprocess.run([SHIM_TEST], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DROPIN), reason="dropin_test not built (needs /root/reference)")
def test_reference_callers_on_b200_dropin():
    r = subprocess.run([DROPIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
