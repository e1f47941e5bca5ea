"""The product's multi-rank data plane across real PROCESSES.

Each case launches P processes (tests/mp_peer_worker.py), one rank each,
rendezvous over gloo on 127.0.0.1, and runs the COVAP sync step through the
C-ABI with steps back to back (no host synchronisation between them):

* peer collective — the send buffers and flag blocks of every rank are
  exported with cudaIpcGetMemHandle and opened by the others
  (covap_peer_export / covap_peer_import, PeerGroup.from_torch_distributed);
  the kernels publish/consume arrival and reduction flags with
  st.release.sys / ld.acquire.sys across processes.  On a one-GPU box the P
  processes share cuda:0 (time-sliced contexts): the memory-ordering and the
  IPC attach are the real cross-process ones, only the link is local.
* NCCL — Communicator.from_torch_distributed + covap_sync_step, one GPU per
  rank (skipped below P devices: NCCL refuses two ranks on one GPU).

Every rank's synchronised gradient, at every step, and its final residual
arena are checked against the rank-ordered oracle mean (trainer.cpp:365-386):
bit for bit for the peer collective (it sums in rank order) and for NCCL at
P <= 2; within |d| <= 1e-6 * sum_w |x_w| / P for NCCL at P > 2.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORKER = os.path.join(ROOT, "tests", "mp_peer_worker.py")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(tmp_path, P, args, timeout=900):
    port = free_port()
    procs, outs = [], []
    for r in range(P):
        out = tmp_path / f"rank{r}.json"
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(P), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, WORKER, "--out", str(out)] + args,
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      start_new_session=True))
        outs.append(out)
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=timeout)[0].decode(errors="replace")[-3000:])
    finally:
        for p in procs:
            if p.poll() is None:
                os.killpg(p.pid, 9)  # the process group this test started
    verdicts = []
    for r, out in enumerate(outs):
        assert out.exists(), f"rank {r} wrote no verdict:\n{logs[r] if r < len(logs) else ''}"
        verdicts.append(json.loads(out.read_text()))
    for v, log in zip(verdicts, logs):
        assert v["ok"], json.dumps(v, indent=1) + "\n" + log
    return verdicts


# (layout, K, P, mode, steps): ResNet-50 K=4 (no sharding), VGG-16 K=4 (fc6 /
# fc7 sharded, the 4 096-element bucket), ResNet-50 K=8 (phases 5-7 empty: the
# same-parity steps 4 and 8 with no collective in between) — in every peer mode.
PEER_CASES = [
    ("resnet50", 4, 2, 1, 5), ("resnet50", 4, 2, 0, 5), ("resnet50", 4, 2, 2, 5),
    ("vgg16", 4, 4, 1, 5), ("vgg16", 4, 4, 0, 3), ("vgg16", 4, 4, 2, 5),
    ("resnet50", 8, 2, 0, 10), ("resnet50", 8, 2, 1, 10), ("resnet50", 8, 3, 2, 10),
    ("resnet50", 1, 4, 1, 2),
]


@pytest.mark.parametrize("layout,K,P,mode,steps", PEER_CASES,
                         ids=[f"{c[0]}-K{c[1]}-P{c[2]}-mode{c[3]}" for c in PEER_CASES])
def test_peer_collective_across_processes(tmp_path, layout, K, P, mode, steps):
    vs = launch(tmp_path, P, ["--collective", "peer", "--layout", layout, "--interval", str(K),
                              "--mode", str(mode), "--steps", str(steps)])
    assert all(v["world"] == P for v in vs)


NCCL_CASES = [("resnet50", 4, 2, 5), ("vgg16", 4, 2, 5), ("resnet50", 8, 2, 10),
              ("resnet50", 4, 4, 5), ("bert_large", 4, 8, 5), ("resnet50", 4, 8, 5)]


@pytest.mark.parametrize("layout,K,P,steps", NCCL_CASES,
                         ids=[f"{c[0]}-K{c[1]}-P{c[2]}" for c in NCCL_CASES])
def test_nccl_sync_across_processes(tmp_path, layout, K, P, steps):
    if torch.cuda.device_count() < P:
        pytest.skip(f"NCCL needs one GPU per rank: {torch.cuda.device_count()} < {P}")
    launch(tmp_path, P, ["--collective", "nccl", "--layout", layout, "--interval", str(K),
                         "--steps", str(steps)])


# The peer kernels over NCCL symmetric-window memory instead of CUDA IPC
# (covap_peer_create_nccl).  P = 1 runs on any box (a 1-rank communicator:
# the window, its peer pointer and the kernels' flag protocol on it); P > 1
# needs one GPU per rank, as NCCL does.  multimem: the reduction in the
# NVSwitch (multimem.ld_reduce / multimem.st), within the NCCL tolerance.
NCCL_PEER_CASES = [("resnet50", 4, 1, 0, False), ("resnet50", 4, 1, 1, False),
                   ("resnet50", 8, 1, 2, False), ("resnet50", 4, 2, 1, False),
                   ("resnet50", 8, 2, 0, False), ("vgg16", 4, 4, 1, False),
                   ("resnet50", 4, 2, 1, True), ("resnet50", 8, 2, 0, True),
                   ("vgg16", 4, 4, 1, True), ("bert_large", 4, 8, 1, True)]


@pytest.mark.parametrize("layout,K,P,mode,mm", NCCL_PEER_CASES,
                         ids=[f"{c[0]}-K{c[1]}-P{c[2]}-mode{c[3]}" + ("-multimem" if c[4] else "")
                              for c in NCCL_PEER_CASES])
def test_peer_over_nccl_window_across_processes(tmp_path, layout, K, P, mode, mm):
    if torch.cuda.device_count() < P:
        pytest.skip(f"NCCL needs one GPU per rank: {torch.cuda.device_count()} < {P}")
    vs = launch(tmp_path, P, ["--collective", "peer_nccl", "--layout", layout, "--interval",
                              str(K), "--mode", str(mode), "--steps", "6"]
                + (["--multimem"] if mm else []))
    assert all(v.get("multimem", False) == mm for v in vs)


def test_peer_multimem_refused_without_multicast(tmp_path):
    """One rank has no NVSwitch multicast team: asking for multimem must fail
    loudly at creation, not fall back."""
    import paper_2311_04499_b200 as covap
    plan = covap.plan_for(covap.load_layout("resnet50"), covap.CovapConfig(interval=4))
    comm = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0)
    state = covap.CompressorState(plan, torch.float32, 0)
    with pytest.raises(covap.Error, match="multicast"):
        covap.PeerGroup.from_nccl(state, comm, multimem=True)
    g = covap.PeerGroup.from_nccl(state, comm)  # the plain window still works
    assert not g.multimem
    del g
    comm.close()
