"""The C++ drop-in (integration/solver_gpu.cpp) written against the
reference's own API: its C++ parity test and the `egsolve solve` equivalent
CLI.  Both binaries are built by the Makefile into oracle/_ref/ (they need
the reference headers) and travel to the GPU box."""
import os
import subprocess

import pytest

from oracle_bindings import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref")
TEST = os.path.join(BIN, "test_solver_gpu")
CLI = os.path.join(BIN, "egsolve_gpu")


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")


def test_dropin_binaries_link():
    for path in (TEST, CLI):
        _need(path)
        out = subprocess.run(["ldd", path], capture_output=True, text=True).stdout
        assert "not found" not in out, out
        assert "libegs_b200.so" in out and "libegsolve_ref.so" in out


@pytest.mark.gpu
def test_cpp_parity_suite():
    _need(TEST)
    r = subprocess.run([TEST], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


@pytest.mark.gpu
def test_cli_solves_spec_fixture(tmp_path):
    _need(CLI)
    f = tmp_path / "g1.eg"
    f.write_text("# SPEC.md G1\neg 2 2\nv 0 0\nv 1 1\ne 0 1 -1\ne 1 0 1\n")
    r = subprocess.run([CLI, str(f)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout == "0 1 1\n1 0\n"
    bad = tmp_path / "bad.eg"
    bad.write_text("eg 2 1\nv 0 0\nv 1 1\ne 0 1 -1\n")  # vertex 1 has no move
    r = subprocess.run([CLI, str(bad)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1


@pytest.mark.gpu
def test_cli_matches_reference_on_c1(tmp_path, reflib, golden):
    _need(CLI)
    a = reflib.fixed(10000, 4, 100, 1)
    f = tmp_path / "c1.eg"
    f.write_text(reflib.write_arena(a))
    r = subprocess.run([CLI, str(f)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    from oracle_bindings import fnv1a64
    rec = golden["fixed/10000/4/100/1"]
    assert f"{fnv1a64(r.stdout.encode()):016x}" == rec["solution_fnv"]
