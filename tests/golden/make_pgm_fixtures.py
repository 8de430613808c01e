"""Copies the reference's CLI fixture pair (proj/tests/data/fixture_3x3*.pgm, used by its
tests/test_cli.cpp:109-120) into tests/golden/ so the GPU-box tests can pin the CLI against it
without /root/reference. Run once where the reference is mounted: python tests/golden/make_pgm_fixtures.py"""
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/proj/tests/data"
for name in ("fixture_3x3.pgm", "fixture_3x3_eroded.pgm"):
    shutil.copyfile(os.path.join(SRC, name), os.path.join(HERE, name))
    print("copied", name, os.path.getsize(os.path.join(HERE, name)), "bytes")
