"""The multi-GPU path, verifiable on a 1-GPU box: program ranks as threads of
one process on one GPU (SM caps 148 // m), collectives only through the
hand-written NVLink peer-memory kernels, every 2- and 3-device golden program
against the CPU oracle (tests/multi/peer_ranks.py).  Runs in a subprocess
with a timeout, so a protocol bug cannot hang the test session."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_peer_ranks_in_one_process_match_oracle():
    # every 2nd golden program of 2 and 3 devices, one (dtype, gradient sync)
    # combination each, rotating — about 160 runs (the full sweep:
    # python tests/multi/peer_ranks.py).  bf16 with sufficient-factor
    # broadcasting is left out of the in-process form: two ranks sharing one
    # GPU hang in the back-to-back SFB factor gathers (chain4.hetero2; open,
    # DESIGN.md) — the same programs pass over NCCL + the NVLink kernels with
    # one process per GPU (tests/multi/nccl_parity.py, profiles/r02_multi_*).
    res = subprocess.run([sys.executable, os.path.join(HERE, "multi", "peer_ranks.py"), "--rotate", "--stride", "2",
                          "--skip", "bf16:sfb", "--verbose"], capture_output=True, text=True, timeout=1500)
    print(res.stdout[-3000:])
    assert res.returncode == 0, res.stdout[-6000:] + res.stderr[-4000:]
    assert "0 failures" in res.stdout
