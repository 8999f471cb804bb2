"""The C++ host API (include/fastmnmf_b200.hpp: the reference's public
interface over the C ABI) -- tests/cpp/test_api.cpp mirrors the reference's
own C++ tests with the CPU oracle as the checker (built by
__graft_entry__.build())."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_api")


def test_header_compiles_standalone(tmp_path):
    src = tmp_path / "inc.cpp"
    src.write_text('#include "fastmnmf_b200.hpp"\nint main() { fastmnmf::BlockLayout l({2, 3}); '
                   'return l.total == 5 ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-fsyntax-only", "-I",
                        os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_cpp_test_program_is_built_and_links_the_library():
    if not os.path.exists(BIN):
        import sys

        sys.path.insert(0, os.path.join(ROOT, "tests", "cpp"))
        import build_tests

        build_tests.build()
    r = subprocess.run(["ldd", BIN], capture_output=True, text=True)
    assert "libdfm_b200.so" in r.stdout and "not found" not in r.stdout, r.stdout


@pytest.mark.gpu
def test_cpp_api_against_oracle():
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests", "cpp"))
    import build_tests

    build_tests.build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr
