"""bench.py itself on the GPU (small shapes): the JSON line keeps the driver's
contract, and the N > 1 path (peer-memory exchange) runs end to end with two
ranks sharing cuda:0 (the build has one GPU)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "e2e", "gpu_launches", "clocks")


def _last_json(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


@pytest.mark.timeout(600)
def test_bench_line_contract_cfg1():
    out = subprocess.run([sys.executable, "bench.py", "--config", "cfg1", "--steps", "5",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True,
                         timeout=580, check=True).stdout
    d = _last_json(out)
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["value"] > 0
    assert d["gpu_launches"] > 0 and d["roofline"]["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * d["config"]["packets_per_slice_per_gpu"]
    assert "cpu_baseline" in d and d["cpu_baseline"]["kind"] == "port"
    # the PCIe ceiling beside e2e: bare pinned copies of the step's H2D + D2H bytes
    pcie = d["e2e"]["pcie"]
    assert pcie["h2d_gbs"] > 0 and pcie["d2h_gbs"] > 0 and pcie["ceiling_value"] > 0
    assert abs(pcie["frac"] - d["e2e"]["value"] / pcie["ceiling_value"]) < 1e-9


@pytest.mark.timeout(600)
def test_bench_two_ranks_share_device_p2p():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                          str(port), "bench.py", "--gpus", "2", "--share-device", "--config",
                          "cfg1", "--steps", "4", "--warmup", "3"], cwd=ROOT, capture_output=True,
                         text=True, timeout=580, check=True).stdout
    d = _last_json(out)
    assert d["n_gpus"] == 2 and d["exchange"]["kind"] == "p2p" and d["value"] > 0
