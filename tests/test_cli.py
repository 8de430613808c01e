"""PGM format and the CLI front end (reference pgm.cpp:55-137,
rectmorph_cli.cpp:105-308, tests/test_pgm.cpp, tests/test_cli.cpp). The format code and the CLI's
argument handling run on CPU; the filtering itself (-m gpu) goes through the GPU library."""
import os
import subprocess

import numpy as np
import pytest

import paper_2002_09474_b200 as pkg
from paper_2002_09474_b200 import build as pbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
CLI = pbuild.CLI


def _cli(*args, timeout=300):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def test_cpp_pgm_binary(tmp_path):
    src = os.path.join(ROOT, "tests", "cpp", "pgm_test.cpp")
    exe = str(tmp_path / "pgm_test")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L", pbuild.PKG, "-lrectmorph_b200", "-lrmgpu", f"-Wl,-rpath,{pbuild.PKG}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "pgm_test ok" in r.stdout, r.stdout + r.stderr


def test_python_pgm_mirror(tmp_path):
    img = (np.arange(35, dtype=np.uint16).reshape(5, 7) * 37 % 256).astype(np.uint8)
    for binary in (True, False):
        data = pkg.write_pgm(img, binary)
        assert np.array_equal(pkg.read_pgm(data), img)
        assert pkg.write_pgm(pkg.read_pgm(data), binary) == data
    assert pkg.write_pgm(np.array([[1, 20], [255, 0]], np.uint8), False) == b"P2\n2 2\n255\n1 20\n255 0\n"
    got = pkg.read_pgm(b"P2 # m\n# c\n2 # w\n1\n255\n5 # p\n6\n")
    assert got.tolist() == [[5, 6]]
    for data, code in [(b"P6\n1 1\n255\nx", pkg.Errc.BadMagic), (b"", pkg.Errc.BadMagic),
                       (b"P5\n0 1\n255\nx", pkg.Errc.BadHeader), (b"P5\n1 1\n254\nx", pkg.Errc.UnsupportedMaxval),
                       (b"P5\n2 2\n255\nab", pkg.Errc.TruncatedData), (b"P2\n1 1\n255\n300\n", pkg.Errc.BadHeader),
                       (b"P2\n2 1\n255\n7\n", pkg.Errc.TruncatedData)]:
        with pytest.raises(pkg.Error) as e:
            pkg.read_pgm(data)
        assert e.value.code == code, data
    path = str(tmp_path / "x.pgm")
    pkg.store_pgm(path, img)
    assert np.array_equal(pkg.load_pgm(path), img)
    with pytest.raises(pkg.Error) as e:
        pkg.load_pgm(str(tmp_path / "absent.pgm"))
    assert e.value.code == pkg.Errc.IoError and "absent.pgm" in str(e.value)
    # the C++ drop-in and the Python mirror write identical bytes
    r = pkg.load_pgm(os.path.join(GOLDEN, "fixture_3x3.pgm"))
    assert pkg.write_pgm(r) == open(os.path.join(GOLDEN, "fixture_3x3.pgm"), "rb").read()


def test_cli_arguments_fail_in_one_line(tmp_path):
    assert os.path.exists(CLI), "build the package first"
    for args in (["--help"], ["apply", "--help"], ["bench", "--help"], ["calibrate", "--help"]):
        rc, out, _ = _cli(*args)
        assert rc == 0 and "usage" in out
    src = os.path.join(GOLDEN, "fixture_3x3.pgm")
    out = str(tmp_path / "o.pgm")
    bad = [[],
           ["frobnicate"],
           ["apply", "--op", "erode", "--se", "3x3", src],
           ["apply", "--op", "shrink", "--se", "3x3", src, out],
           ["apply", "--op", "erode", "--se", "4x3", src, out],
           ["apply", "--op", "erode", "--se", "3", src, out],
           ["apply", "--op", "erode", "--se", "3x3", "--border", "mirror", src, out],
           ["apply", "--op", "erode", "--se", "3x3", "--border", "constant:300", src, out],
           ["apply", "--op", "erode", "--se", "3x3", "--config", str(tmp_path / "none.cfg"), src, out],
           ["apply", "--op", "erode", "--se", "3x3", str(tmp_path / "missing.pgm"), out],
           ["bench", "--windows", "3..9:3", "--out", str(tmp_path / "b.csv")],
           ["bench", "--windows", "9..3", "--out", str(tmp_path / "b.csv")],
           ["calibrate", "--windows", "2..8", "--out", str(tmp_path / "c.cfg")],
           ["calibrate", "--windows", "3..9", "--out", str(tmp_path / "c.cfg"), "--reps", "0"]]
    for args in bad:
        rc, so, se = _cli(*args)
        assert rc == 1, args
        assert se.startswith("rectmorph:") and se.count("\n") == 1, (args, se)
    assert not os.path.exists(out)


@pytest.mark.gpu
def test_cli_apply_fixture_and_ops(gpu, restatement, tmp_path):
    # the reference's fixture pair (its test_cli.cpp:109-120): byte-identical output
    out = str(tmp_path / "eroded.pgm")
    rc, so, se = _cli("apply", "--op", "erode", "--se", "3x3", "--border", "replicate",
                      os.path.join(GOLDEN, "fixture_3x3.pgm"), out)
    assert rc == 0 and so == "" and se == "", se
    assert open(out, "rb").read() == open(os.path.join(GOLDEN, "fixture_3x3_eroded.pgm"), "rb").read()
    # every op and both borders against the oracle on a random image
    img = restatement.generate(97, 61, 77)
    src = str(tmp_path / "in.pgm")
    pkg.store_pgm(src, img, binary=False)
    ops = {"erode": 0, "dilate": 1, "open": 2, "close": 3, "gradient": 4}
    for name, op in ops.items():
        for border, (mode, val) in (("replicate", (0, 0)), ("constant:17", (1, 17))):
            dst = str(tmp_path / f"{name}.pgm")
            rc, _, se = _cli("apply", "--op", name, "--se", "9x5", "--border", border, src, dst)
            assert rc == 0, se
            assert np.array_equal(pkg.load_pgm(dst), restatement.morph(img, 9, 5, op, mode, val)), (name, border)
    # a calibrated config steers the planner, never the pixels
    cfgs = {"lin": "threshold_h=127\nthreshold_v=127\nsource=calibrated\n",
            "vh": "threshold_h=1\nthreshold_v=1\nsource=calibrated\n"}
    outs = []
    for tag, text in cfgs.items():
        cfg = str(tmp_path / f"{tag}.cfg")
        open(cfg, "w").write(text)
        dst = str(tmp_path / f"d_{tag}.pgm")
        assert _cli("apply", "--op", "dilate", "--se", "41x33", "--config", cfg, src, dst)[0] == 0
        outs.append(open(dst, "rb").read())
    assert outs[0] == outs[1]
    assert np.array_equal(pkg.read_pgm(outs[0]), restatement.morph(img, 41, 33, 1))


@pytest.mark.gpu
def test_cli_bench_and_calibrate(gpu, tmp_path):
    csv = str(tmp_path / "b.csv")
    rc, _, se = _cli("bench", "--width", "512", "--height", "256", "--windows", "3..15:4", "--reps", "3",
                     "--transpose", "--out", csv)
    assert rc == 0, se
    lines = open(csv).read().splitlines()
    assert lines[0] == "axis,algorithm,window,image_w,image_h,reps,median_ns,device_median_ns"
    assert len(lines) == 1 + 4 * 4 + 1
    for ln in lines[1:-1]:
        axis, algo, w, iw, ih, reps, ns, dns = ln.split(",")
        assert axis in ("horizontal", "vertical") and algo in ("linear", "vanherk") and int(ns) > 0 and int(dns) > 0
    cfg = str(tmp_path / "c.cfg")
    rc, so, se = _cli("calibrate", "--width", "256", "--height", "128", "--windows", "3..11", "--reps", "3",
                      "--out", cfg)
    assert rc == 0, se
    parsed = pkg.load_config(cfg)
    assert parsed.source == "calibrated" and so == pkg.format_config(parsed)
