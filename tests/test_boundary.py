"""The drop-in boundary, checked without a GPU: the C-ABI library loads and
exports every symbol include/*.h declares; the Python mirror of the reference
API validates arguments like the reference (vexsort.cpp:19-31)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2205_05982_b200 as vx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            src = open(os.path.join(inc, f)).read()
            syms |= set(re.findall(r"\b(vxs_[a-z_0-9]+)\s*\(", src))
    return syms


def test_library_exports_every_declared_symbol():
    lib = vx.lib()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(vx.EXPORTED_SYMBOLS) == syms


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {vx.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_host_only_queries():
    assert vx.lib().vxs_version().startswith(b"vxsort_b200")
    for kt, b in vx.KEY_BYTES.items():
        assert vx.lib().vxs_key_bytes(vx.KEY_CODE[kt]) == b
    assert vx.base_case_capacity("u64") >= 4096
    ws = vx.workspace_bytes(100_000_000, "u64")
    assert 800_000_000 <= ws < 1_200_000_000  # temp keys + O(n/cap) scheduler state
    assert vx.workspace_bytes(0, "u32") > 0


def test_invalid_arguments_map_to_value_error():
    lib = vx.lib()
    st = vx.SortStats()
    # unknown key type / order -> VXS_INVALID_ARGUMENT without touching a GPU
    assert lib.vxs_sort(None, 0, 42, 0, 0, 0, None, 0, None, ctypes.byref(st)) == 1
    assert lib.vxs_sort(None, 0, 3, 7, 0, 0, None, 0, None, ctypes.byref(st)) == 1
    assert lib.vxs_sort(None, 5, 3, 0, 0, 0, None, 0, None, ctypes.byref(st)) == 1
    assert b"NULL" in lib.vxs_last_error()
    with pytest.raises(ValueError):
        vx.sort(np.zeros(4, np.uint64), vx.SortConfig(scratch=vx.SortScratch(16)))
    with pytest.raises(ValueError):
        vx.sort(np.zeros((4, 2), np.uint64))  # K128 needs an explicit key type
    with pytest.raises(ValueError):
        vx.sort(np.zeros(4, np.complex64))
    # a 2-D array of a 1-word key type is rejected, not sorted by its first column
    with pytest.raises(ValueError):
        vx.sort(np.zeros((4, 3), np.int32), key_type="i32")
    with pytest.raises(ValueError):
        vx.sort(np.zeros((4, 3), np.uint64), key_type="k128")
    with pytest.raises(ValueError):
        vx.sort(np.zeros((), np.uint32), key_type="u32")


def test_dist_create_validates_the_group():
    """vxs_dist_create rejects bad groups before touching a device."""
    from paper_2205_05982_b200.dist import _ALLGATHER_FN, _DistGroup
    lib = vx.lib()
    out = ctypes.c_void_p()
    for rank, world in ((0, 0), (2, 2), (-1, 1)):
        g = _DistGroup(rank, world, None, _ALLGATHER_FN(0), None)
        assert lib.vxs_dist_create(ctypes.byref(g), ctypes.byref(out)) == 1
    g = _DistGroup(0, 2, None, _ALLGATHER_FN(0), None)  # world > 1 needs NCCL or a host all-gather
    assert lib.vxs_dist_create(ctypes.byref(g), ctypes.byref(out)) == 1
    assert b"allgather" in lib.vxs_last_error()
    assert lib.vxs_dist_sort(None, None, 0, 6, 0, 1, 0, ctypes.byref(out), ctypes.byref(ctypes.c_size_t()),
                             None, None) == 1


def test_trivial_host_sorts_need_no_device():
    # n <= 1 returns before touching the device (driver.hpp:175)
    for n in (0, 1):
        x = np.arange(n, dtype=np.uint32)
        st = vx.sort(x)
        assert st.max_depth == 0 and st.partition_calls == 0


def test_cpp_header_mirrors_reference_surface():
    hpp = open(os.path.join(ROOT, "include", "vexsort_b200.hpp")).read()
    for t in ("std::int16_t", "std::uint16_t", "std::int32_t", "std::uint32_t", "float",
              "std::int64_t", "std::uint64_t", "double", "K128"):
        assert re.search(r"SortStats sort\(std::span<%s> keys" % re.escape(t), hpp), t
    for name in ("struct SortConfig", "class SortScratch", "scratch_bytes", "enum class Order",
                 "enum class Backend", "wide_backend_is_simd"):
        assert name in hpp


def test_cpp_dropin_compiles_links_and_runs(tmp_path):
    """INTEGRATION.md's recompile-only drop-in: a reference-style call site
    (harness.cpp:264 / test_driver.cpp style) compiles against
    include/vexsort_b200.hpp, links libvxsort_b200.so, and runs the
    device-free paths (n <= 1, too-small scratch -> std::invalid_argument)."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    src = tmp_path / "dropin.cpp"
    src.write_text(r'''
#include <cstdio>
#include <vector>
#include "vexsort_b200.hpp"
int main() {
  std::vector<std::uint64_t> one{42};
  vexsort::SortStats st = vexsort::sort(std::span<std::uint64_t>(one), vexsort::SortConfig{});
  if (st.max_depth != 0 || one[0] != 42) return 1;
  std::vector<float> none;
  vexsort::sort(std::span<float>(none));
  std::vector<vexsort::K128> k(1);
  vexsort::sort(std::span<vexsort::K128>(k), vexsort::SortConfig{.order = vexsort::Order::kDescending});
  vexsort::SortScratch small(16);
  std::vector<std::int32_t> v{3, 1, 2};
  try {
    vexsort::SortConfig cfg;
    cfg.scratch = &small;
    vexsort::sort(std::span<std::int32_t>(v), cfg);
    return 2;
  } catch (const std::invalid_argument&) {
  }
  if (false) {  // instantiate the device-pointer entry points
    vexsort::sort_device<std::uint32_t>(nullptr, 0);
    vexsort::argsort_device<std::uint32_t>(nullptr, 0, nullptr);
    vexsort::sort_pairs_device<std::int64_t, double>(nullptr, nullptr, 0);
  }
  std::puts("ok");
  return 0;
}
''')
    exe = tmp_path / "dropin"
    lib_dir = os.path.join(ROOT, "paper_2205_05982_b200", "lib")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                        "-L", lib_dir, "-lvxsort_b200", f"-Wl,-rpath,{lib_dir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.returncode, r.stdout, r.stderr)
