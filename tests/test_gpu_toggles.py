"""The non-default kernel paths behind environment toggles (read once per
process by libadaptra) re-run the stage F / B / W parity suites (small and
full-size) in a fresh process: one grouped column-sum launch instead of one per
sum, one dW launch per product instead of the grouped GEMM, epilogue
inputs by LDG instead of TMA, no W pairs, the ping-pong attention forward (opt-in), 2x2-cluster GEMMs
with the A tile multicast (opt-in), half of the attention forward's
exponentials on the FMA pipe (ex2_poly), bias gradients by separate
column-sum launches instead of inside the grouped dW launch.  (The P-in-TMEM
attention variants -- ptmem, qtmem, sep, s2 -- passed these suites in
profiles/r02_attn_*_ab.jsonl but are not run here: an intermittent hang under
the 8-stage bench keeps them experimental.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("toggle", [{"ADAPTRA_COLSUM_GROUPED": "1"},
                                    {"ADAPTRA_GEMM_GROUPED": "0"},
                                    {"ADAPTRA_EPI_IN_LDG": "1"},
                                    {"ADAPTRA_W_PAIRS": "0"},
                                    {"ADAPTRA_W_GROUP": "2"},
                                    {"ADAPTRA_ATTN_FWD": "pp"},
                                    {"ADAPTRA_GEMM_MC": "1"},
                                    {"ADAPTRA_ATTN_POLY": "2"},
                                    {"ADAPTRA_DB_FUSED": "0"}])
def test_stage_parity_under_toggle(toggle):
    env = dict(os.environ, **toggle)
    files = ["tests/test_gpu_stage.py", "tests/test_gpu_fullsize.py"]
    if "ADAPTRA_W_PAIRS" in toggle or "ADAPTRA_W_GROUP" in toggle:   # executor toggles: pipelined iterations
        files = ["tests/test_gpu_pipeline.py"]
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider"] + [
        os.path.join(ROOT, f) for f in files]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert " passed" in r.stdout and "failed" not in r.stdout
