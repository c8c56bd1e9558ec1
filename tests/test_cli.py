"""The CLI (paper_2003_06324_b200/_lib/fireiron): the reference's ctest
entries (proj/tests/CMakeLists.txt:24-36) re-run against the B200 backend."""
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT

CLI = os.path.join(ROOT, "paper_2003_06324_b200", "_lib", "fireiron")
L2 = os.path.join(GOLDEN, "listings", "listing2.fi")


def run(*args, timeout=300):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout)


def test_cli_elaborate_and_codegen(tmp_path):
    r = run("elaborate", os.path.join(GOLDEN, "listings", "listing1.fi"))
    assert r.returncode == 0 and len(r.stdout.splitlines()) == 12
    out = tmp_path / "k.cu"
    r = run("codegen", L2, "--out", str(out))
    assert r.returncode == 0 and "fi_fma_unfused" in out.read_text()


def test_cli_rejects_bad_override():  # cli_rejects_bad_override (WILL_FAIL)
    r = run("verify", L2, "--m", "100")
    assert r.returncode == 1 and "NonDivisible" in r.stderr


@pytest.mark.gpu
def test_cli_verify_listing2():  # cli_verify_listing2
    r = run("verify", L2, "--seed", "7")
    assert r.returncode == 0 and r.stdout.startswith("PASS max_error=0 ")


@pytest.mark.gpu
def test_cli_verify_override():  # cli_verify_override
    r = run("verify", L2, "--m", "256", "--n", "256", "--seed", "9")
    assert r.returncode == 0 and r.stdout.startswith("PASS")


@pytest.mark.gpu
def test_cli_simulate_digest_matches_reference():
    r = run("simulate", L2, "--seed", "7")
    assert r.returncode == 0 and "digest=0xaa6d3cc65c6c7b67" in r.stdout


@pytest.mark.gpu
def test_cli_simulate_rejects_hmma():  # cli_simulate_rejects_hmma (WILL_FAIL)
    assert run("simulate", os.path.join(GOLDEN, "listings", "hmma_ptx.fi")).returncode == 1


@pytest.mark.gpu
def test_cli_matrix_io_roundtrip(tmp_path):  # cli_matrix_io
    mv = os.path.join(GOLDEN, "listings", "move_identity.fi")
    a, b = tmp_path / "io1.txt", tmp_path / "io2.txt"
    assert run("simulate", mv, "--seed", "4", "--dump-c", str(a)).returncode == 0
    assert run("simulate", mv, "--load-a", str(a), "--dump-c", str(b)).returncode == 0
    assert a.read_text() == b.read_text()


@pytest.mark.gpu
def test_cli_verify_tensor_core_strategy(tmp_path):
    import paper_2003_06324_b200 as fi
    s = tmp_path / "tc.fi"
    s.write_text(fi.strategies.tc_strategy(512, 512, 256))
    r = run("verify", str(s), "--seed", "3")
    assert r.returncode == 0 and "backend=tcgen05" in r.stdout and r.stdout.startswith("PASS max_error=0 ")


def test_cli_check_async(tmp_path, fi):  # CPU protocol check of the tcgen05 launch
    f = tmp_path / "c3.fi"
    f.write_text(fi.strategies.c3_strategy())
    r = run("check-async", str(f))
    assert r.returncode == 0 and r.stdout.startswith("async protocol check: ok")
    assert "slices 4 + remainder" in r.stdout
    r = run("check-async", L2)  # FMA-leaf tree: no tcgen05 lowering
    assert r.returncode == 1 and "InvalidTree" in r.stderr
