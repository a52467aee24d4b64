"""The ringsim-compatible CLI: config schema, exit codes and the volume
report match the reference (CPU); verify / profile / compare on the GPU."""

import io
import json
import os

import pytest

from conftest import ROOT, load_json
from paper_2412_20501_b200 import cli
from paper_2412_20501_b200.errors import ConfigError

CFG = os.path.join(ROOT, "configs")


def write(tmp_path, data):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(data))
    return str(p)


BASE = {"problem": {"seq_len": 64, "heads": 2, "head_dim": 16, "causal": True, "seed": 1},
        "parallel": {"ranks": 4, "nodes": 1}, "schedule": {"kind": "zigzag-token-ring"}}


def test_volume_matches_reference_output():
    gold = load_json("cli_volume.json")
    assert set(gold) == set(os.listdir(CFG))
    for name, text in gold.items():
        buf = io.StringIO()
        assert cli.cmd_volume(cli.load_config(os.path.join(CFG, name)), out=buf) == 0
        assert buf.getvalue() == text, name


@pytest.mark.parametrize("mutate,msg", [
    (lambda d: d.update(extra={}), "unknown config section"),
    (lambda d: d["problem"].update(dtype="bf16"), "unknown key"),
    (lambda d: d["problem"].update(causal=False), "requires causal=true"),
    (lambda d: d["problem"].update(seq_len=60), "2P must divide seq_len"),
    (lambda d: d["schedule"].update(kind="hybrid"), "hybrid schedule requires causal=false"),
    (lambda d: (d["schedule"].update(kind="hybrid"), d["problem"].update(causal=False),
                d["parallel"].update(nodes=3)), "nodes must divide ranks"),
    (lambda d: d["schedule"].update(kind="bogus"), "unknown schedule kind"),
    (lambda d: d.update(topology={"kind": "torus"}), "unknown topology kind"),
    (lambda d: d.update(timing={"efficiency": 1.5}), "efficiency"),
    (lambda d: d["parallel"].update(ranks=0), "ranks must be a positive integer"),
])
def test_config_validation(mutate, msg):
    data = json.loads(json.dumps(BASE))
    mutate(data)
    with pytest.raises(ConfigError, match=msg):
        cli.RunConfig.from_dict(data)


def test_token_ring_rejects_causal():
    data = json.loads(json.dumps(BASE))
    data["schedule"]["kind"] = "token-ring"
    with pytest.raises(ConfigError, match="requires causal=false"):
        cli.RunConfig.from_dict(data)


def test_exit_codes(tmp_path, capsys):
    bad = write(tmp_path, {"problem": {}})
    assert cli.main(["volume", "--config", bad]) == 2
    assert cli.main(["volume", "--config", str(tmp_path / "missing.json")]) == 3
    assert cli.main(["volume", "--config", write(tmp_path, BASE)]) == 0
    assert cli.main(["bogus"]) == 2


def test_parse_sweep():
    assert cli.parse_sweep("seq_len=4096..32768") == ("seq_len", [4096, 8192, 16384, 32768])
    with pytest.raises(ConfigError):
        cli.parse_sweep("heads=1..4")


def test_switch_model_charges_ports():
    cfg = cli.RunConfig.from_dict(json.loads(json.dumps(BASE)))
    sched = cli.build_schedule(cfg)
    send, recv = cli.modelled_comm(cfg, sched)
    assert len(send) == sched.n_steps and all(len(r) == 4 for r in send)
    assert max(send[0]) > 0 and max(recv[-1]) > 0


@pytest.mark.gpu
def test_verify_profile_compare_on_gpu(tmp_path, capsys):
    assert cli.main(["verify", "--config", os.path.join(CFG, "example_verify.json")]) == 0
    assert "status=PASS" in capsys.readouterr().out
    assert cli.main(["verify", "--config", write(tmp_path, BASE)]) == 0
    t, s = tmp_path / "t.json", tmp_path / "s.csv"
    assert cli.main(["profile", "--config", write(tmp_path, BASE), "--trace", str(t),
                     "--summary", str(s)]) == 0
    events = json.loads(t.read_text())
    assert {e["tid"] for e in events} <= {"compute", "send", "recv"}
    assert all(e["ph"] == "X" and isinstance(e["ts"], int) for e in events)
    lines = s.read_text().splitlines()
    assert lines[0] == cli.SUMMARY_HEADER and lines[-1].split(",")[5] == "total"
    capsys.readouterr()
    data = json.loads(json.dumps(BASE))
    data["problem"]["causal"] = False
    data["schedule"]["kind"] = "token-ring"
    assert cli.main(["compare", "--config", write(tmp_path, data), "--schedules",
                     "ring,token-ring", "--sweep", "seq_len=64..128"]) == 0
    rows = capsys.readouterr().out.splitlines()
    assert rows[0] == cli.COMPARE_HEADER and len(rows) == 5


def _reference_ringsim():
    """The reference package (baseline/_ref install, else its source tree), or None."""
    import importlib
    import sys
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "ringsim")):
            if path not in sys.path:
                sys.path.append(path)
            try:
                return importlib.import_module("ringsim.cli"), importlib.import_module("ringsim.netsim")
            except Exception:
                return None
    return None


@pytest.mark.parametrize("cfg_name,override", [
    ("a10_token_ring.json", None), ("a10_ring.json", None),
    ("a10_token_ring.json", {"kind": "ring", "bandwidth_gbps": 50.0, "latency_us": 3.0}),
    ("a10_ring.json", {"kind": "switch", "bandwidth_gbps": 900.0, "latency_us": 5.0}),
    ("a10_ring.json", {"kind": "full-mesh", "bandwidth_gbps": 25.0, "latency_us": 5.0})])
def test_modelled_comm_equals_reference_netsim(cfg_name, override):
    """The modelled send/recv lanes equal the reference's netsim.simulate
    (outbound / inbound per step and rank) on the reference's own configs --
    including its fitted A10 matrix topology -- and on ring / switch /
    full-mesh variants of them."""
    ref = _reference_ringsim()
    if ref is None:
        pytest.skip("reference package not available")
    rcli, rnet = ref
    from paper_2412_20501_b200 import cli
    path = os.path.join(ROOT, "configs", cfg_name)
    if not os.path.exists(path):
        path = os.path.join("/root/reference/pkg/configs", cfg_name)
    if not os.path.exists(path):
        pytest.skip("config not available")
    data = json.load(open(path))
    if override:
        data["topology"] = override
    mine = cli.RunConfig.from_dict(json.loads(json.dumps(data)))
    theirs = rcli.RunConfig.from_dict(json.loads(json.dumps(data)))
    send, recv = cli.modelled_comm(mine, cli.build_schedule(mine))
    from ringsim.engine import trace_from_schedule
    tl = rnet.simulate(trace_from_schedule(rcli.build_schedule(theirs)),
                       rcli.build_topology(theirs), rcli.build_timing(theirs))
    import numpy as np
    assert np.allclose(np.array(send), tl.outbound, rtol=1e-12, atol=0)
    assert np.allclose(np.array(recv), tl.inbound, rtol=1e-12, atol=0)
