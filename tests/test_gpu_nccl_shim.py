"""GPU: fastusp's NCCL backend (NcclComm: ncclCommInitRank, ncclCommSplit, grouped
ncclSend/ncclRecv, ncclCommGetAsyncError / ncclCommAbort) executing at world 2 and 4.

Real NCCL refuses two ranks on one GPU and this build reaches a single B200, so the ranks are
threads of one process and libnccl is replaced at load time by tests/nccl_shim (LD_PRELOAD):
a test-only NCCL with the same point-to-point contract over copy-engine pulls.  Everything
above the NCCL calls -- fastusp's mesh split, wire layouts, pipelined ring, LSE all-to-all,
sub-group communicators, async-error polling and abort -- is the product code.  Checks:
  * usp_attention at (N,R) in {(2,1),(2,2),(4,2),(4,4),(4,1)}, bf16 and FP8, against the oracle,
    BIT-identical to the same layer over the in-process fabric, identical TrafficLog bytes;
  * ulysses / ring over world-split sub-groups (fusp_group_create -> ncclCommSplit);
  * a peer that never joins: DeadlockError (fabric.hpp:112) and aborted communicators.
Eager only: the shim's host rendezvous cannot be graph-captured."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SHIM = os.path.join(HERE, "nccl_shim", "_build", "libnccl_shim.so")


def run(which):
    if not os.path.exists(SHIM):
        subprocess.run(["make", "-C", os.path.join(HERE, "nccl_shim")], check=True)
    env = dict(os.environ, LD_PRELOAD=SHIM, FUSP_SHIM_TIMEOUT_S="4")
    p = subprocess.run([sys.executable, os.path.join(HERE, "nccl_shim", "drive.py"), which],
                       capture_output=True, text=True, timeout=900, env=env)
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert lines, p.stderr[-3000:]
    return lines, p


def test_nccl_backend_usp_world_2_and_4(cuda, fu):
    lines, p = run("usp")
    assert len(lines) == 6, p.stderr[-2000:]
    bad = [x for x in lines if not x["ok"]]
    assert not bad, bad


def test_nccl_backend_subgroups(cuda, fu):
    lines, p = run("groups")
    assert all(x["ok"] for x in lines), (lines, p.stderr[-2000:])


def test_nccl_dead_peer_raises_deadlock(cuda, fu):
    lines, p = run("dead")
    assert all(x["ok"] for x in lines), (lines, p.stderr[-2000:])


def test_nccl_backend_peer_windows(cuda, fu):
    lines, p = run("peer")
    assert len(lines) == 3 and all(x["ok"] for x in lines), (lines, p.stderr[-2000:])
