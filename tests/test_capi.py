"""CPU suite for the boundary: the C-ABI library loads, exports every symbol include/rmgpu.h
declares, validates arguments exactly like the reference before touching a device, and the
C++ drop-in library exports the reference's entry points. No kernel runs here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2002_09474_b200 as pkg
from paper_2002_09474_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header: str) -> set[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    return set(re.findall(r"^\s*(?:int|void|const char\*|unsigned long long)\s+(rmgpu_\w+)\s*\(", text, re.M))


def test_library_exports_every_declared_symbol():
    declared = _declared("rmgpu.h")
    assert len(declared) >= 25
    L = pkg.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rmgpu_\w+)", out))
    assert declared <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_abi_basics():
    L = pkg.lib()
    assert L.rmgpu_abi_version() == 1
    assert L.rmgpu_status_string(2) == b"EvenExtent"
    # resolve: Auto -> Linear iff window <= threshold, inclusive (dispatch.cpp:14-20)
    assert pkg.resolve(pkg.PassAlgorithm.Auto, 69, pkg.Axis.Horizontal) == pkg.PassAlgorithm.Linear
    assert pkg.resolve(pkg.PassAlgorithm.Auto, 71, pkg.Axis.Horizontal) == pkg.PassAlgorithm.VanHerk
    assert pkg.resolve(pkg.PassAlgorithm.Auto, 59, pkg.Axis.Vertical) == pkg.PassAlgorithm.Linear
    assert pkg.resolve(pkg.PassAlgorithm.Auto, 61, pkg.Axis.Vertical) == pkg.PassAlgorithm.VanHerk
    assert pkg.resolve(pkg.PassAlgorithm.VanHerk, 3, pkg.Axis.Vertical) == pkg.PassAlgorithm.VanHerk


def test_validation_before_any_device_work():
    L = pkg.lib()
    nul = C.c_void_p(0)
    # even / zero extents (make_se, image.cpp:18-24): checked before pointers or the device
    assert L.rmgpu_morph_u8(nul, 16, nul, 16, 4, 4, 4, 3, 0, 0, 0, 0, 0, nul) == 2
    assert L.rmgpu_morph_u8(nul, 16, nul, 16, 4, 4, 3, 0, 0, 0, 0, 0, 0, nul) == 1
    assert L.rmgpu_morph_u16(nul, 16, nul, 16, 4, 4, 0, 2, 0, 0, 0, 0, 0, nul) == 1  # zero wins over even
    # negative sizes -> BadArgument (Image::Image, image.cpp:28-29)
    assert L.rmgpu_morph_u8(nul, 16, nul, 16, -1, 4, 3, 3, 0, 0, 0, 0, 0, nul) == 11
    # empty images are a no-op
    assert L.rmgpu_morph_u8(nul, 16, nul, 16, 0, 4, 3, 3, 0, 0, 0, 0, 0, nul) == 0
    # bad op / border / constant out of range
    assert L.rmgpu_morph_u8(nul, 16, nul, 16, 4, 4, 3, 3, 9, 0, 0, 0, 0, nul) == 11
    assert L.rmgpu_morph_u8(nul, 16, nul, 16, 4, 4, 3, 3, 0, 1, 256, 0, 0, nul) == 11
    # unsupported tile side (transpose.cpp:7-10)
    for n in (0, 2, 5, 32):
        assert L.rmgpu_transpose_tiles_u8(nul, 1, n, n, n * n, nul) == 3
    assert L.rmgpu_window_1d_u8(nul, 10, 4, 0, 0, 0, 1, nul, nul) == 2
    assert L.rmgpu_pass_u8(0, nul, 16, nul, 16, 4, 4, -1, 0, 0, 0, 0, nul) == 1
    assert b"odd" in L.rmgpu_last_error() or b">= 1" in L.rmgpu_last_error()


def test_python_mirror_errors():
    with pytest.raises(pkg.Error) as e:
        pkg.make_se(4, 3)
    assert e.value.code == pkg.Errc.EvenExtent
    with pytest.raises(pkg.Error) as e:
        pkg.make_se(3, 0)
    assert e.value.code == pkg.Errc.ZeroExtent
    with pytest.raises(pkg.Error) as e:
        pkg.linear_window_1d(np.zeros(4, np.uint8), 2, pkg.OpKind.Erode)
    assert e.value.code == pkg.Errc.EvenExtent
    with pytest.raises(pkg.Error) as e:
        pkg.transpose_tile(np.zeros(25, np.uint8), 5, 5)
    assert e.value.code == pkg.Errc.UnsupportedTile


def test_plan_names():
    assert pkg.plan_name(1, 100, 100, 1, 1) == "copy"
    assert pkg.plan_name(1, 4096, 4096, 3, 3) != ""


def test_cpp_dropin_library_exports_reference_api():
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", _native.HOSTLIB_PATH], capture_output=True,
                         text=True).stdout
    for sym in ["rectmorph::erode(", "rectmorph::dilate(", "rectmorph::opening(", "rectmorph::closing(",
                "rectmorph::gradient(", "rectmorph::transpose_image(", "rectmorph::transpose_tile(",
                "rectmorph::horizontal_pass(", "rectmorph::vertical_pass_direct(",
                "rectmorph::vertical_pass_via_transpose(", "rectmorph::morph_separable(",
                "rectmorph::linear_window_1d(", "rectmorph::van_herk_1d(", "rectmorph::resolve(",
                "rectmorph::make_se(", "rectmorph::format_config", "rectmorph::parse_config(",
                "rectmorph::load_config(", "rectmorph::save_config(", "rectmorph::calibrate("]:
        assert sym in out, sym


def test_no_cpu_fallback_in_product():
    # the product package must not import the oracle or run numpy morphology
    src = ""
    for root, _, files in os.walk(os.path.join(ROOT, "paper_2002_09474_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                src += open(os.path.join(root, f)).read()
    assert "import oracle" not in src and "from oracle" not in src
    assert "liboracle" not in src and "librmref" not in src


# ---- dispatch config + calibrate (dispatch.hpp:46-66): host-only, no device ------------------
def test_config_text_round_trip_and_grammar():
    cfg = pkg.DispatchConfig(33, 101, "calibrated")
    text = pkg.format_config(cfg)
    assert text == "threshold_h=33\nthreshold_v=101\nsource=calibrated\n"
    assert pkg.parse_config(text) == cfg
    assert pkg.format_config(pkg.DispatchConfig()) == "threshold_h=69\nthreshold_v=59\nsource=paper\n"
    got = pkg.parse_config("# comment\n\nthreshold_h = 69\nthreshold_v=59\r\nsource= paper\n")
    assert got == pkg.DispatchConfig(69, 59, "paper")
    for bad in ["threshold_h=69\nthreshold_v=59\n",
                "threshold_h=69\nthreshold_v=59\nsource=paper\nextra=1\n",
                "threshold_h=68\nthreshold_v=59\nsource=paper\n",
                "threshold_h=-3\nthreshold_v=59\nsource=paper\n",
                "threshold_h=abc\nthreshold_v=59\nsource=paper\n",
                "threshold_h=69\nthreshold_h=69\nthreshold_v=59\nsource=paper\n",
                "threshold_h=69\nthreshold_v=59\nsource=guessed\n",
                "threshold_h 69\nthreshold_v=59\nsource=paper\n"]:
        with pytest.raises(pkg.Error) as e:
            pkg.parse_config(bad)
        assert e.value.code == pkg.Errc.BadConfig, bad
    with pytest.raises(pkg.Error) as e:
        pkg.parse_config("threshold_h=69\nthreshold_v=59\nsource=guessed\n")
    assert "line 3" in str(e.value)


def test_config_files(tmp_path):
    cfg = pkg.DispatchConfig(45, 91, "calibrated")
    path = str(tmp_path / "dispatch.txt")
    pkg.save_config(path, cfg)
    assert open(path).read() == "threshold_h=45\nthreshold_v=91\nsource=calibrated\n"
    assert pkg.load_config(path) == cfg
    with pytest.raises(pkg.Error) as e:
        pkg.load_config(str(tmp_path / "missing.txt"))
    assert e.value.code == pkg.Errc.IoError and "missing.txt" in str(e.value)


def test_calibrate_validates_before_the_device():
    for args, code in [((32, 32, [3, 5], 2), pkg.Errc.InsufficientReps),
                       ((32, 32, [5, 3], 3), pkg.Errc.BadArgument),
                       ((32, 32, [3, 4], 3), pkg.Errc.EvenExtent),
                       ((32, 32, [], 3), pkg.Errc.BadArgument),
                       ((0, 32, [3], 3), pkg.Errc.BadArgument)]:
        with pytest.raises(pkg.Error) as e:
            pkg.calibrate(*args)
        assert e.value.code == code, args


def test_cpp_config_binary(tmp_path):
    # the reference's config API, compiled against the drop-in header and run without a GPU
    src = os.path.join(ROOT, "tests", "cpp", "config_test.cpp")
    exe = str(tmp_path / "config_test")
    pkgdir = os.path.join(ROOT, "paper_2002_09474_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L", pkgdir, "-lrectmorph_b200", "-lrmgpu", f"-Wl,-rpath,{pkgdir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "config_test ok" in r.stdout
