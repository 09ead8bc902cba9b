"""Build tests/c_abi_test.c with gcc -std=c11 against include/gemm_f16.h and the
in-tree libgemm_f16.so: a plain-C client of the boundary (no C++, no Python)."""
import os
import subprocess

import pytest

import paper_2108_13191_b200 as g

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _build(tmp_path):
    g.load_library()
    libdir = os.path.dirname(g.library_path())
    exe = str(tmp_path / "c_abi_test")
    cmd = ["gcc", "-std=c11", "-Wall", "-Werror", "-pedantic", os.path.join(HERE, "c_abi_test.c"),
           "-I", os.path.join(ROOT, "include"), "-L", libdir, "-l:libgemm_f16.so", f"-Wl,-rpath,{libdir}",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_client_argument_handling(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "c_abi_test OK" in r.stdout


@pytest.mark.gpu
def test_c_client_gemm_on_device(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_abi_test OK (gpu)" in r.stdout


def test_options_struct_layout_matches_header(tmp_path):
    # the Python binding's ctypes mirror of gemm_options_t must agree with the C header
    # field by field (size and every offset), or options land in the wrong member
    fields = [name for name, _ in g._Options._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include "gemm_f16.h"\nint main(void) {\n'
                   '  printf("size %zu\\n", sizeof(gemm_options_t));\n'
                   + "".join(f'  printf("{f} %zu\\n", offsetof(gemm_options_t, {f}));\n' for f in fields)
                   + "  return 0;\n}\n")
    exe = str(tmp_path / "layout")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", str(src), "-I", os.path.join(ROOT, "include"), "-o", exe],
                   check=True, capture_output=True, text=True)
    got = dict(line.split() for line in subprocess.run([exe], capture_output=True, text=True, check=True)
               .stdout.splitlines())
    import ctypes
    assert int(got["size"]) == ctypes.sizeof(g._Options)
    for f in fields:
        assert int(got[f]) == getattr(g._Options, f).offset, f
