"""CLI commands that need no GPU (planner, usage errors), against the
reference's CLI contract (test_cli.py:184-250)."""

import json

import numpy as np
import pytest

from paper_2502_15443_b200.cli import main
from paper_2502_15443_b200.latency import REFERENCE_PROFILE, Architecture, CompressionPlan, HardwareProfile, latency


def run(capsys, *argv):
    code = main([str(a) for a in argv])
    out = capsys.readouterr()
    return code, out.out, out.err


def test_simulate_matches_latency_function(tmp_path, capsys):
    plan = CompressionPlan.block_plan(16 * 2**20, 24, 3)
    p = tmp_path / "plan.json"
    p.write_text(plan.to_json())
    code, out, _ = run(capsys, "simulate", "--plan", p, "--cr", 1.7, "--arch", "gpu_buffer", "--json")
    assert code == 0
    doc = json.loads(out)
    want = latency(REFERENCE_PROFILE, plan, Architecture.GPU_BUFFER, np.where(plan.compressed_mask, 1.7, 1.0))
    assert doc["per_sample_latency"] == want.per_sample_latency
    assert doc["bottleneck"] == want.bottleneck.value and doc["stage_seconds"] == want.stage_seconds


def test_profile_and_plan_files(tmp_path, capsys):
    prof, plan = tmp_path / "profile.json", tmp_path / "plan.json"
    prof.write_text(REFERENCE_PROFILE.to_json())
    plan.write_text(CompressionPlan.block_plan(16 * 2**20, 78, 2).to_json())
    code, out, _ = run(capsys, "simulate", "--profile", prof, "--plan", plan, "--cr", 1.8, "--arch", "auto", "--json")
    assert code == 0 and json.loads(out)["per_sample_latency"] > 0
    assert HardwareProfile.from_json(prof.read_text()) == REFERENCE_PROFILE
    code, out, _ = run(capsys, "simulate", "--profile", prof, "--n-chunks", 10, "--json")
    assert code == 0
    json.loads(out)
    code, out, _ = run(capsys, "simulate", "--n-chunks", 10)
    assert code == 0 and out.startswith("architecture: ")


def test_simulate_budget(capsys):
    code, out, err = run(capsys, "simulate", "--n-chunks", 40, "--cr", 2.0, "--budget", 1e9)
    assert code == 0 and "block_size: 1" in out and err == ""
    code, out, err = run(capsys, "simulate", "--n-chunks", 40, "--cr", 2.0, "--budget", 1e-12)
    assert code == 0 and "block_size: 0" in out and "infeasible" in err
    code, _, err = run(capsys, "simulate", "--budget", 1.0)
    assert code == 3 and "--n-chunks" in err
    code, _, err = run(capsys, "simulate")
    assert code == 3


def test_usage_error_exit_2(capsys):
    with pytest.raises(SystemExit) as exc:
        main(["quantize"])
    assert exc.value.code == 2


def test_synth_bytes_equal_reference_cli(tmp_path, capsys):
    """synth writes exactly the files the reference's `dcomp synth` writes
    (sha256 recorded from the reference CLI in tests/golden/cli_synth.json),
    and prints the same text."""
    import hashlib
    import os

    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "cli_synth.json")) as f:
        want = json.load(f)
    w, s = tmp_path / "w.dcwt", tmp_path / "s.json"
    code, out, _ = run(capsys, "synth", "--out-weights", w, "--out-stats", s, "--seed", 0)
    assert code == 0 and out.splitlines()[0] == "attn_q: 512x512" and out.splitlines()[-1].startswith("wrote 6 tensors")
    assert hashlib.sha256(w.read_bytes()).hexdigest() == want["w.dcwt"]
    assert hashlib.sha256(s.read_bytes()).hexdigest() == want["s.json"]
    assert run(capsys, "synth", "--out-weights", w, "--out-stats", s, "--preset", "single", "--rows", 64,
               "--cols", 32, "--name", "t", "--seed", 3)[0] == 0
    assert hashlib.sha256(w.read_bytes()).hexdigest() == want["w1.dcwt"]
    assert hashlib.sha256(s.read_bytes()).hexdigest() == want["s1.json"]
