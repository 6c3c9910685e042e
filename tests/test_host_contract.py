"""CPU checks of the host-side contract: the bench's reference arm (the oracle timed on the host)
prints one well-formed JSON line, and the user-spectra generator produces what the f4 tests need."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np

import oracle as O
import synth

ROOT = Path(__file__).resolve().parents[1]


def test_bench_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "images/s"
    assert d["config"]["workload"] == "config1"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_random_spectra_generator():
    n, eta = 32, 9
    g = synth.random_spectra(n, eta, 4)
    assert g.shape == (eta, n, n) and np.all(g >= 0)
    assert O.frame_tightness(g) < 1e-14
    neg = (n - np.arange(n)) % n                    # -u on the centred grid
    d = g - g[:, neg][:, :, neg]
    assert np.max(np.abs(d[:, 1:, 1:])) == 0.0     # point-symmetric off the Nyquist lines
    assert np.max(np.abs(d)) > 0.0                  # asymmetric on them
    h = n // 2
    assert np.all(g[0] > 0)                         # plane 0 covers the grid
    cols = [np.nonzero(np.any(g[i] != 0, axis=0))[0] - h for i in range(1, eta)]
    assert any(len(c) < n for c in cols)            # some planes are pruned to column bands
    assert np.array_equal(g, synth.random_spectra(n, eta, 4))
