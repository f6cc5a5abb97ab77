"""bench.py host logic on CPU: the reference arm's JSON line (contract keys, every requested step timed, the GPU
arm's config dict) with the oracle run stubbed out -- no oracle arithmetic is exercised here (tests/test_oracle_pins.py
does that); the non-zero ranks of a torchrun launch exit without work."""
import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402
from oracle import ckks, plan  # noqa: E402


class _StubOracle:
    """OracleArgmax with the (13 s) circuit replaced by a fixed time: the parameter set, layout and plan are real."""
    calls = 0

    def __init__(self):
        self.plan = plan
        self.lay = synth.LAYOUTS["argmax_k2"]
        self.ev = types.SimpleNamespace(prm=ckks.Params(synth.PARAM_SETS["argmax"]))

    def run(self):
        _StubOracle.calls += 1
        return 0.5, self.lay["queries"], 4


def _args(**kw):
    a = types.SimpleNamespace(gpus=1, steps=7, warmup=3, batch=16, ref_warmup=False)
    a.__dict__.update(kw)
    return a


def test_reference_arm_line(monkeypatch, capsys):
    monkeypatch.setattr(bench, "OracleArgmax", _StubOracle)
    monkeypatch.delenv("RANK", raising=False)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    _StubOracle.calls = 0
    bench.run_reference(_args())
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["steps"] == 7 and line["steps_requested"] == 7 and _StubOracle.calls == 7  # no warm-up runs by default
    assert line["higher_is_better"] is True and line["vs_baseline"] is None and line["n_gpus"] == 1
    assert abs(line["value"] - 2048 / 0.5) < 1e-6 and abs(line["ms_per_step"] - 500.0) < 1e-6
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 4 and cb["value"] == line["value"] and "7 of 7" in cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": bench.UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the GPU arm's config for the same --batch: 16 ciphertexts of 2 x 30 limbs, 6 Galois keys + the relinearisation key
    prm = ckks.Params(synth.PARAM_SETS["argmax"])
    n_rot = len(plan.argmax_rotations(synth.LAYOUTS["argmax_k2"]))
    want = bench.workload_config(16, 1, 2048, 2 * prm.nq * prm.N, n_rot, prm.nq, prm.np_, prm.alpha, prm.N)
    assert line["config"] == want and want["workload"] == bench.WORKLOAD
    assert "503 MB ciphertexts" in want["l2"] and want["parallelism"] == "single GPU"


def test_reference_arm_cap_and_other_ranks(monkeypatch, capsys):
    monkeypatch.setattr(bench, "OracleArgmax", _StubOracle)
    monkeypatch.setattr(bench, "REF_CAP_S", 1.2)  # 0.5 s stub steps: the third step crosses the cap
    monkeypatch.delenv("RANK", raising=False)
    bench.run_reference(_args(steps=10))
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["steps"] == 3 and line["steps_requested"] == 10 and "capped" in line["cpu_baseline"]["sample"]
    # under torchrun only rank 0 runs the oracle; the others print nothing
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    _StubOracle.calls = 0
    bench.run_reference(_args())
    assert capsys.readouterr().out == "" and _StubOracle.calls == 0
