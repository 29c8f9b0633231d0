"""Multi-GPU NCCL grid parity (needs >= 2 GPUs; skipped on a 1-GPU box)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _gpus():
    from paper_2202_09512_b200 import _lib
    return _lib.device_count()


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
@pytest.mark.parametrize("nproc", [2, 4])
def test_grid_matches_oracle(nproc, exchange):
    """exchange='peer': the per-iteration exchange runs over peer memory
    (peer.cuh) wherever the dense K in {16, 32} path applies; 'nccl': RK_PEER=0
    keeps the NCCL collectives."""
    if _gpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc + (10 if exchange == "nccl" else 0)),
           os.path.join(ROOT, "tools", "grid_check.py")]
    env = dict(os.environ, RK_PEER="1" if exchange == "peer" else "0")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert out.returncode == 0 and line, out.stdout[-2000:] + out.stderr[-2000:]
    rep = json.loads(line[-1])
    assert rep["ok"], rep
    used = {c.get("exchange") for c in rep["cases"] if c["engine"] != "sparse" and c["k"] in (16, 32)}
    assert used == {exchange}, rep


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
@pytest.mark.parametrize("nproc", [2, 4])
def test_grid_cfg3_block_matches_oracle(nproc, exchange):
    """cfg3's n = 32768, k = 32 on the 1x2 / 2x2 grid: solve_on_grid with a
    per-rank BlockSource vs the fp64 oracle (tools/grid_check_big.py)."""
    if _gpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + nproc + (10 if exchange == "nccl" else 0)),
           os.path.join(ROOT, "tools", "grid_check_big.py")]
    env = dict(os.environ, RK_PEER="1" if exchange == "peer" else "0")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert out.returncode == 0 and line, out.stdout[-2000:] + out.stderr[-2000:]
    rep = json.loads(line[-1])
    assert rep["ok"] and rep["exchange"] == exchange, rep
