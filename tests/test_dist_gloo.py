"""CPU, world_size 2 and 4 over gloo: the host-side logic of the one-process-per-GPU path.

* NCCL unique-id distribution, max-over-ranks timing and sequence sharding
  (paper_2602_10940_b200.dist, used by bench.py under torchrun);
* each rank's mesh groups agree with the C ABI's make_mesh and across ranks;
* a rehearsal of the USP layer's wire protocol with the exact slot layouts libfastusp.so
  uses (Ulysses slot t = [Q|K|V] head block t; output slot t = rows t*S/N of our heads;
  ring K/V hop to (pos+1) mod R), exchanged with real inter-process all_to_all / send-recv
  and checked against the reference oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, r, fp8, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import restate as R
    from oracle.make_golden import qkv
    from paper_2602_10940_b200 import dist as fdist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        # uid broadcast + max over ranks
        uid = fdist.broadcast_bytes(bytes(range(128)) if rank == 0 else None)
        assert uid == bytes(range(128))
        assert fdist.max_over_ranks(rank + 1.5) == world + 0.5
        # mesh groups: the same on every member, equal to the C ABI's make_mesh
        ug, rg = fdist.mesh_groups(world, r, rank)
        try:
            import paper_2602_10940_b200 as fu
            m = fu.make_mesh(world, r)
            assert m.ulysses_group(rank).members == ug and m.ring_group(rank).members == rg
        except FileNotFoundError:
            pass
        allg = [None] * world
        dist.all_gather_object(allg, (ug, rg))
        for other, (oug, org) in enumerate(allg):
            if other in ug:
                assert oug == ug
            if other in rg:
                assert org == rg

        # wire-protocol rehearsal (H=8, S=64, D=128)
        h, s, d = 8, 64, 128
        q, k, v = qkv((1, h, s, d), (1, h, s, d))
        u = world // r
        hp, sl = h // u, s // world
        rows = fdist.shard_rows(s, world, rank)
        lq, lk, lv = (x[:, :, rows] for x in (q, k, v))
        if fp8:
            lk, lv = R.fake_quant(lk), R.fake_quant(lv)
        # Ulysses in: slot t = heads [t*hp,(t+1)*hp) of Q|K|V (usp.cpp ulysses_in / pack_kernel)
        send = np.stack([np.concatenate([x[:, t * hp:(t + 1) * hp].ravel() for x in (lq, lk, lv)])
                         for t in range(u)]).astype(np.float32)
        recv = np.empty_like(send)
        if u > 1:
            # all_to_all within the Ulysses group: emulate with a world-size exchange
            full_send = np.zeros((world,) + send.shape[1:], np.float32)
            for t, m_ in enumerate(ug):
                full_send[m_] = send[t]
            full_recv = np.empty_like(full_send)
            dist.all_to_all_single(torch.from_numpy(full_recv), torch.from_numpy(full_send))
            recv = np.stack([full_recv[m_] for m_ in ug])
        else:
            recv = send
        blk = hp * sl * d
        span = u * sl
        Qr = np.concatenate([recv[j, :blk].reshape(1, hp, sl, d) for j in range(u)], axis=2)
        Kr = np.concatenate([recv[j, blk:2 * blk].reshape(1, hp, sl, d) for j in range(u)], axis=2)
        Vr = np.concatenate([recv[j, 2 * blk:].reshape(1, hp, sl, d) for j in range(u)], axis=2)
        # ring: hop i receives the chunk from position (pos - i) mod R (protocols.cpp:253-257)
        pos = rg.index(rank)
        o, l = R.attention_with_lse(Qr, Kr, Vr)
        o, l = o.astype(np.float32), l.astype(np.float32)
        ck, cv = Kr, Vr
        for i in range(1, r):
            sk, sv = (R.fake_quant(ck), R.fake_quant(cv)) if fp8 else (ck, cv)
            nk, nv = np.empty_like(sk), np.empty_like(sv)
            nxt, prv = rg[(pos + 1) % r], rg[(pos - 1) % r]
            reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(sk)), nxt),
                    dist.isend(torch.from_numpy(np.ascontiguousarray(sv)), nxt)]
            dist.recv(torch.from_numpy(nk), prv)
            dist.recv(torch.from_numpy(nv), prv)
            for q_ in reqs:
                q_.wait()
            ck, cv = nk, nv
            po, pl = R.attention_with_lse(Qr, ck, cv)
            o, l = R.merge_lse(o, l, po.astype(np.float32), pl.astype(np.float32))
        # Ulysses out: slot t = our heads over rows [t*sl,(t+1)*sl) (attention epilogue layout)
        osend = np.stack([o[:, :, t * sl:(t + 1) * sl].ravel() for t in range(u)])
        if u > 1:
            full_send = np.zeros((world, osend.shape[1]), np.float32)
            for t, m_ in enumerate(ug):
                full_send[m_] = osend[t]
            full_recv = np.empty_like(full_send)
            dist.all_to_all_single(torch.from_numpy(full_recv), torch.from_numpy(full_send))
            orecv = np.stack([full_recv[m_] for m_ in ug])
        else:
            orecv = osend
        mine = np.concatenate([orecv[j].reshape(1, hp, sl, d) for j in range(u)], axis=1)
        want = R.usp_attention(q, k, v, world, r, fp8=fp8)[:, :, rows]
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.abs(mine - want).max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,r,fp8", [(2, 1, False), (2, 2, False), (2, 2, True),
                                          (4, 2, False), (4, 2, True), (4, 4, False)])
def test_gloo_multiprocess_protocol(tmp_path, world, r, fp8):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, r, fp8, str(tmp_path)), nprocs=world, join=True)
    errs = [float(np.load(tmp_path / f"rank{i}.npy")) for i in range(world)]
    assert max(errs) < 1e-5, errs
