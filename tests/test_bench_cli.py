"""bench.py's host-side contract on CPU: --gpus N outside torchrun re-launches
itself under torch.distributed.run with N local ranks (127.0.0.1 rendezvous,
NCCL init logging on stderr); the record helpers."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    sys.path.insert(0, ROOT)
    import importlib
    return importlib.import_module("bench")


def test_self_launch_command(monkeypatch):
    bench = _bench()
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--workload", "cfg3"])
    args = bench.parse()
    assert bench.self_launch(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--workload", "cfg3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
    assert seen["env"]["NCCL_DEBUG_FILE"] == "/dev/stderr"


def test_main_dispatches_self_launch_without_torchrun_env(monkeypatch):
    bench = _bench()
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    monkeypatch.setattr(bench, "self_launch", lambda args: 7)
    try:
        bench.main()
    except SystemExit as e:
        assert e.code == 7
    else:
        raise AssertionError("main() did not exit with the launcher's status")


def test_trig_hash_and_traffic_lookup(tmp_path, monkeypatch):
    bench = _bench()
    from paper_2212_09460_b200 import synth
    c, s = synth.q15_table(180)
    h1 = bench.trig_hash(c, s)
    c2 = c.copy()
    c2[5] += 1
    assert h1 != bench.trig_hash(c2, s) and len(h1) == 64
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "ncu_traffic.json").write_text(json.dumps(
        {"cfg3": {"hough_vote_pairs_kernel<2>": 123456}}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.ncu_traffic("cfg3", "hough_vote_pairs_kernel") == 123456
    assert bench.ncu_traffic("cfg4", "hough_vote_pairs_kernel") is None
    assert isinstance(bench.host_info()["nproc"], int)
    assert np.isfinite(bench.hbm_peak_gbs())
