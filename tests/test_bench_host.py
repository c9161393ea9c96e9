"""Host-side checks of bench.py (no GPU): the reference arm's JSON line (the oracle timed on the
host cores, the contract's `--impl reference` leg) and the pure helpers behind the roofline
numbers — the whole-step roof of SURVEY §8(d) item 8 and the profile-tag → kernel map."""
import importlib.util
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_step_roofline_matches_survey_formula():
    b = _bench()
    N, E, B, A = 1000.0, 40000.0, 8000.0, 60000.0
    flops, byts, t_tensor, t_hbm = b.step_roofline((N, E, B, A), "3xtf32")[:4]
    assert flops == pytest.approx(3.0 * (286592 * E + 380800 * A + 28544 * B + 75136 * N))
    assert byts == pytest.approx(3.0 * (256 * (14 * E + 6 * A + 7 * B + 12 * N) + 24 * E + 12 * A))
    assert t_tensor == pytest.approx(flops / (b.tensor_peak("3xtf32") * 1e12))
    assert t_hbm == pytest.approx(byts / (b.PEAKS["hbm_gbs"] * 1e9))
    # the 3xTF32 roof is a third of the TF32 one; BF16 is the measured bf16 peak
    assert b.tensor_peak("3xtf32") == pytest.approx(b.tensor_peak("tf32") / 3.0)
    assert b.tensor_peak("bf16") > b.tensor_peak("tf32")


def test_kernel_of_maps_tensor_core_tags():
    b = _bench()
    assert b.kernel_of("ac_f1", "3xtf32") == "k_rowgemm_tc"
    assert b.kernel_of("ac_f1", "fp32") == "k_rowgemm"
    assert b.kernel_of("segsum_bc_S", "3xtf32") == "k_segsum"
    assert b.PREC_CODE == {"fp32": 0, "3xtf32": 1, "tf32": 2, "bf16": 3}


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    """`bench.py --impl reference` runs the oracle (fp64, CPU) on the bench workload and prints ONE
    JSON line with the contract's keys (impl, metric, value, e2e with zero copies, cpu_baseline)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "structures/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["steps"] == 1 and d["warmup"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["config"]["workload"] == "C2"
