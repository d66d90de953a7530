"""One rank of the cross-process peer-memory test (tests/test_gpu_peer.py): a separate process
on cuda:0 whose window reaches the other rank's through CUDA IPC (cudaIpcGetMemHandle /
cudaIpcOpenMemHandle), as one-process-per-GPU ranks do over NVLink.  Handles travel through
files in a scratch directory (the caller's own bootstrap: fusp_ctx_peer_window / _open).
usage: python tests/peer_ipc_worker.py RANK WORLD DIR [RING_DIM FP8 GRAPH BATCH]
(FP8: 0 off, 1 per tensor, 2 per (b,h) block)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_10940_b200 as fu  # noqa: E402
from oracle import restate as R  # noqa: E402
from oracle.make_golden import qkv  # noqa: E402


def wait_for(path, timeout=120.0):
    t0 = time.time()
    while not os.path.exists(path):
        if time.time() - t0 > timeout:
            raise TimeoutError(path)
        time.sleep(0.01)


def main():
    rank, world, d = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    r = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    fp8 = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    graph = len(sys.argv) > 6 and sys.argv[6] == "1"
    bsz = int(sys.argv[7]) if len(sys.argv) > 7 else 1
    torch.cuda.set_device(0)
    h, s = 8, 256 * world
    probs = [qkv((bsz, h, s, 128), (bsz, h, s, 128), seeds=(600 + i, 610 + i, 620 + i)) for i in range(3)]
    mesh = fu.make_mesh(world, r)
    opts = fu.CommOptions(fp8_kv=fp8 > 0, fp8_block=int(fp8 == 2), pipelined_ring=True,
                          check_finite=False, out_dtype=torch.float32)
    # a fabric of `world` ranks of which this process runs one: the peer path at R = 1 moves
    # every byte through the windows, the fabric is never entered
    fab = fu.Fabric(world)
    ctx = fu.WorkerContext.local(fab, rank, 0)
    wb = fu.peer_window_bytes(world, r, (bsz, h, s // world, 128), torch.bfloat16, opts)
    mine = ctx.peer_window(wb)
    tmp = os.path.join(d, f"h{rank}.tmp")
    with open(tmp, "wb") as f:
        f.write(mine)
    os.rename(tmp, os.path.join(d, f"h{rank}"))
    handles = []
    for r in range(world):
        wait_for(os.path.join(d, f"h{r}"))
        with open(os.path.join(d, f"h{r}"), "rb") as f:
            handles.append(f.read())
    ctx.peer_open(handles)
    outs = []
    shs = [[torch.from_numpy(np.ascontiguousarray(R.split_sequence(t, world)[rank])).cuda().bfloat16()
            for t in p] for p in probs]
    stream = torch.cuda.Stream()  # (graph capture needs a stream other than the legacy one)
    with torch.cuda.stream(stream):
        for sh in shs:
            outs.append(fu.usp_attention(ctx, *sh, mesh, opts).clone())
        gouts = []
        if graph:  # the same three layers as ONE CUDA graph: ring hops and reshards inside
            qkv3 = [torch.stack([sh[t] for sh in shs]) for t in range(3)]
            y = torch.empty(3, *shs[0][0].shape, device="cuda", dtype=torch.float32)
            g = fu.LayerGraph(ctx, *qkv3, y, mesh, opts, 3)
            for _ in range(3):  # back-to-back replays reuse every window buffer
                g.launch()
            gouts = [y[i].clone() for i in range(3)]
            outs.append(fu.usp_attention(ctx, *shs[0], mesh, opts).clone())  # eager after replays
        ctx.synchronize(timeout_s=60)
        if graph:
            g.close()
    stats = ctx.peer_stats()
    torch.save({"outs": [o.cpu() for o in outs], "gouts": [o.cpu() for o in gouts], "stats": stats},
               os.path.join(d, f"out{rank}.pt"))
    # keep the window mapped until every rank has finished reading / writing it
    open(os.path.join(d, f"done{rank}"), "w").close()
    for r in range(world):
        wait_for(os.path.join(d, f"done{r}"))
    ctx.close()
    fab.close()


if __name__ == "__main__":
    main()
