"""The C ABI from plain C: include/doa.h compiles as C99 (CPU) and examples/doa_demo runs the
hot path on device-generated frames and finds the true DOAs (GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_is_c99():
    src = "#include \"doa.h\"\nint main(void) { doa_plan_t p = 0; (void)p; return (int)DOA_OK; }\n"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-pedantic", "-fsyntax-only", "-I",
                        os.path.join(ROOT, "include"), "-x", "c", "-"], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["music", "mn"])
def test_c_demo_finds_the_sources(alg):
    import __graft_entry__
    exe = __graft_entry__.build_demo()
    r = subprocess.run([exe, alg, "16", "4", "2048", "256", "0.01"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    m = re.search(r"worst \|error\| ([0-9.]+) deg, missing (\d+)", r.stdout)
    assert m, r.stdout
    assert float(m.group(1)) < 0.5 and int(m.group(2)) == 0, r.stdout
