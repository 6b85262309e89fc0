"""Topology probe on the GPU box: real NVML data for cuda:0.
A B200 in an HGX/DGX baseboard has its NVLink 5 ports on NVSwitches, so the
probe reports the switch model (one-hop trees)."""
import json
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_probe_reports_the_nvswitch_model_from_nvml():
    import paper_1910_04940_b200 as B
    import subprocess
    bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", "0"],
                         capture_output=True, text=True).stdout.strip()
    d = B.topology_json([bus])
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "probe_gpu0.json"), "w") as f:
        json.dump({"bus_id": bus, "probe": d}, f)
    assert d["kind"] in ("nvswitch", "pcie"), d
    if d["kind"] == "nvswitch":
        assert d["switch_ports"][0] >= 1
    # a comm over two virtual ranks on cuda:0 reports the probe in its plan
    comms = B.init_all([0, 0])
    assert comms[0].plan(True, 0, 1024, "f32")["topology"]["kind"] == "virtual"
    for c in comms:
        c.destroy()
