"""The command-line front end (paper_2309_16682_b200/cli.py) against the
reference tool's contract (proj/tools/vmt19937_main.cpp, proj/tests/test_cli.cpp):
usage errors exit 2, the bench CSV checksum equals the reference's
run_benchmark checksum, `stat` reproduces the reference's reports, `jump`
writes the reference's bytes."""
import hashlib
import subprocess
import sys

import pytest

from conftest import ROOT

import paper_2309_16682_b200.cli as cli


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2309_16682_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("args", [[], ["frobnicate"], ["bench", "--format", "xml"], ["jump", "-o", "x"],
                                  ["stat", "--tests", "monobit,nope"], ["stat", "--tests", ","],
                                  ["bench", "--generator", "scalar", "-M", "4"],
                                  ["bench", "--generator", "scalar", "--block", "16"],
                                  ["bench", "--block", "7"]])
def test_usage_errors_exit_2(args):
    assert cli.main(args) == cli.EXIT_USAGE


def test_stat_auto_exponent():
    # main.cpp:158-165
    assert cli.stat_auto_exponent(10_000_000, 4) == 22
    assert cli.stat_auto_exponent(1000, 4) == 10
    assert cli.stat_auto_exponent(4_000_000, 4) == 20


def test_self_test_all_fail(golden):
    """--self-test on the constant 0xDEADBEEF source: every test fails (exit 1),
    with the reference's statistics (host-only path, no GPU needed)."""
    r = run("stat", "--self-test", "-n", "1000000")
    assert r.returncode == 1, r.stderr
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 3 and all(line.rstrip().endswith("FAIL") for line in lines)
    ref = golden["stats"]["self_test_0xDEADBEEF"]
    assert f"stat={ref[0]['statistic']:<14.6g}".strip() in lines[0]
    assert f"stat={ref[1]['statistic']:<14.6g}".strip() in lines[1]


@pytest.mark.gpu
def test_bench_csv_checksums_match_reference(golden):
    for row in golden["bench_checksums"]:
        if row["mode"] != 2:
            continue
        r = run("bench", "-M", str(row["lanes"]), "--block", "state", "-n", str(row["count"]),
                "--jump-exponent", str(row["q"]), "--format", "csv")
        assert r.returncode == 0, r.stderr
        f = r.stdout.strip().split(",")
        assert f[0] == "vmt" and int(f[1]) == row["lanes"] and int(f[3]) == row["count"]
        assert int(f[6], 16) == row["xor"], row


@pytest.mark.gpu
def test_stat_reports_match_reference(golden):
    c = [x for x in golden["stats"]["reports"] if x["lanes"] == 4 and x["q"] == 20][0]
    r = run("stat", "-M", "4", "-n", str(c["count"]), "--tests", "monobit,chi2", "--jump-exponent", "20")
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.strip().splitlines()
    assert f"stat={c['monobit']['statistic']:<14.6g}".strip() in lines[0]
    assert f"stat={c['chi2_bytes']['statistic']:<14.6g}".strip() in lines[1]


@pytest.mark.gpu
def test_jump_command_writes_reference_bytes(golden, tmp_path):
    out = str(tmp_path / "F_2p16.vmtj")
    r = run("jump", "-q", "16", "-o", out)
    assert r.returncode == 0, r.stderr
    with open(out, "rb") as f:
        assert hashlib.sha256(f.read()).hexdigest() == golden["vmtj"]["16"]["sha256"]
    # and bench/stat accept it (exponent adopted; a contradicting request fails)
    r = run("bench", "-M", "8", "-n", "100000", "--jump-matrix", out, "--format", "csv")
    assert r.returncode == 0, r.stderr
    r = run("bench", "-M", "8", "-n", "100000", "--jump-matrix", out, "--jump-exponent", "3")
    assert r.returncode == 1 and "holds exponent 16" in r.stderr
