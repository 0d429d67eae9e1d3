"""CLI plumbing on CPU (gen-qc / convert / usage errors) and on the GPU (decode, sweep)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2507_10424_b200.cli", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=600)


def test_gen_qc_and_convert_idempotent(tmp_path):
    a, b, c = tmp_path / "h.alist", tmp_path / "h2.alist", tmp_path / "h3.alist"
    assert run("gen-qc", "--row-blocks", "2", "--col-blocks", "4", "--z", "7", "--out", str(a)).returncode == 0
    assert run("convert", "--in", str(a), "--out", str(b)).returncode == 0
    assert run("convert", "--in", str(b), "--out", str(c)).returncode == 0
    assert a.read_text() == b.read_text() == c.read_text()
    assert a.read_text().splitlines()[0] == "28 14"


def test_usage_and_data_errors(tmp_path):
    assert run().returncode == 1
    assert run("decode").returncode == 1
    bad = tmp_path / "bad.alist"
    bad.write_text("3 1\n1 9\n")
    assert run("convert", "--in", str(bad), "--out", str(tmp_path / "o")).returncode == 2


@pytest.mark.gpu
def test_decode_and_sweep(tmp_path):
    from gen import codes

    h = tmp_path / "p.alist"
    h.write_text(codes.to_alist(codes.paper_5x10()))
    llr = tmp_path / "r.txt"
    llr.write_text("\n".join(["-1", "-1", "0.4"] + ["-1"] * 7) + "\n")
    r = run("decode", "--matrix", str(h), "--llr", str(llr))
    assert r.returncode == 0 and r.stdout.strip() == "isCodeword=1 k=1 b=0000000000"  # worked example P4
    out = tmp_path / "s.csv"
    r = run("sweep", "--matrix", str(h), "--snr", "1,3", "--frames", "2000", "--out", str(out), "--timings")
    assert r.returncode == 0, r.stderr
    assert any(ln.startswith("resident ") for ln in r.stderr.splitlines()), r.stderr  # stage-timing table
    lines = out.read_text().splitlines()
    assert lines[0] == "snr_db,frames,raw_ber,decoded_ber,fer,avg_iterations,wall_seconds,throughput_bps"
    assert len(lines) == 3 and all(len(x.split(",")) == 8 for x in lines)


def test_scaling_usage():
    assert run("scaling", "--gpus", "0").returncode == 1


@pytest.mark.gpu
def test_scaling_one_gpu(tmp_path):
    """scalingStudy on the GPUs this box has (1 here): one row per visible count, outcomes consistent."""
    out = tmp_path / "sc.csv"
    r = run("scaling", "--config", "c1", "--gpus", "1", "--steps", "1", "--warmup", "3", "--out", str(out))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "gpus,wall_seconds,throughput_bps,frames,sum_iterations,frame_errors,bit_errors"
    assert len(lines) == 2 and lines[1].startswith("1,") and int(lines[1].split(",")[3]) == 10000
