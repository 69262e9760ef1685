"""The C ABI library loads and exports every symbol include/vdi.h declares;
host-only helpers (no GPU) behave as documented."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, golden


def _header_functions():
    src = open(os.path.join(ROOT, "include", "vdi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(vdi_[a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def L():
    from paper_2206_14503_b200 import _lib
    return _lib


def test_exports_every_declared_symbol(L):
    names = _header_functions()
    assert len(names) >= 15, names
    lib = C.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"libvdi.so does not export {n}"
    # and the binding declares exactly the header's functions
    assert sorted(L.SIGNATURES) == names


def test_sm100a_code_present(L):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_helpers(L):
    lib = L.lib()
    b, e = C.c_uint32(), C.c_uint32()
    # strips of a 1080-row image on 8 ranks: 135 rows each (Q13)
    for g in range(8):
        assert lib.vdi_strip_rows(1080, 8, g, C.byref(b), C.byref(e)) == 0
        assert (b.value, e.value) == (135 * g, 135 * (g + 1))
    # balanced split of 10 rows on 3 ranks
    sizes = []
    for g in range(3):
        lib.vdi_strip_rows(10, 3, g, C.byref(b), C.byref(e))
        sizes.append(e.value - b.value)
    assert sorted(sizes, reverse=True) == golden("primitives.json")["partition"]["sizes"]
    assert lib.vdi_strip_rows(10, 3, 3, C.byref(b), C.byref(e)) != 0
    # block placement of PEs
    assert [lib.vdi_pe_home(8, 4, p) for p in range(8)] == [0, 0, 1, 1, 2, 2, 3, 3]
    assert [lib.vdi_pe_home(16, 8, p) for p in range(16)] == [p // 2 for p in range(16)]
    assert [lib.vdi_pe_home(8, 1, p) for p in range(8)] == [0] * 8
    # full representation size: 1920x1080, k=20 -> 949.2 MiB of slots + counts
    g = golden("primitives.json")["full_rep_size"]
    fb = lib.vdi_full_bytes(1920, 1080, 20)
    assert fb - 1920 * 1080 == g["W"] * g["H"] * g["k"] * g["bytes_per_slot"]
    assert lib.vdi_status_string(6) == b"VDI_ERR_CAPACITY"
    assert lib.vdi_version().startswith(b"libvdi")


def test_init_rejects_bad_config(L):
    lib = L.lib()
    h = C.c_void_p()

    def cfg(**kw):
        d = dict(width=64, height=64, k_in=4, k_out=4, n_pes=2, n_ranks=1, rank=0, root=0, max_iters=0, gamma_max=0.0,
                 flags=0, nccl_unique_id=None, cuda_stream=None)
        d.update(kw)
        return L.vdi_config(**d)

    for bad in (dict(k_out=0), dict(k_in=256), dict(n_pes=0), dict(n_pes=65), dict(rank=1),
                dict(n_ranks=2, rank=1), dict(root=1), dict(width=0), dict(n_ranks=100, height=64)):
        c = cfg(**bad)
        assert lib.vdi_composite_init(C.byref(c), C.byref(h)) == 1, bad  # VDI_ERR_INVALID_ARG
        assert lib.vdi_last_error(None)
    lib.vdi_composite_destroy(None)  # NULL-safe


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2206_14503_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f


def test_header_is_plain_c_and_links(tmp_path):
    """include/vdi.h compiles as C99 (no C++ in the boundary) and a C program
    links against libvdi.so and calls its host-only entry points."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2206_14503_b200", "lib")
    if not os.path.exists(os.path.join(libdir, "libvdi.so")):
        pytest.skip("libvdi.so not built")
    src = tmp_path / "abi.c"
    src.write_text(r"""
#include <stdio.h>
#include "vdi.h"
int main(void) {
  uint32_t a = 0, b = 0;
  if (vdi_strip_rows(1080, 8, 3, &a, &b) != VDI_OK || a != 405 || b != 540) return 1;
  if (vdi_strip_rows(1080, 8, 8, &a, &b) == VDI_OK) return 2;          /* g >= n_ranks: an error */
  if (vdi_pe_home(16, 8, 15) != 7) return 3;
  if (vdi_full_bytes(1920, 1080, 20) != (uint64_t)1920 * 1080 * (1 + 24 * 20)) return 4;
  if (!vdi_version() || !vdi_status_string(VDI_ERR_INVALID_ARG)) return 5;
  printf("%s\n", vdi_version());
  return 0;
}
""")
    exe = tmp_path / "abi"
    r = subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"), str(src), "-o", str(exe),
                        "-L", libdir, "-lvdi", "-Wl,-rpath," + libdir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
