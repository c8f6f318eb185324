"""Partitioned (multi-rank) path, host side: partition, local meshes with
ghosts, send/recv lists, and the partitioned RHS through a 2-rank gloo
exchange on the CPU (numpy kernel model) against the global oracle."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, build_mesh, set_random_materials

import oracle
from paper_1507_02557_b200.partition import build_local_parts, partition_elements


@pytest.mark.parametrize("method", ["xslab", "rcb"])
def test_send_recv_lists_consistent(method):
    from paper_1507_02557_b200.mesh import structured_hybrid_mesh
    m = structured_hybrid_mesh(4, nx=8)
    parts = build_local_parts(m, partition_elements(m, 3, method))
    total = {t: 0 for t in m.elem_types}
    for p in parts:
        for t in p.types:
            total[t] += p.n_owned[t]
            own = p.global_ids[t][:p.n_owned[t]]
            assert len(set(own.tolist())) == len(own)
        for s, per_t in p.send.items():
            for t, idx in per_t.items():
                a, b = parts[s].recv[p.rank][t]
                np.testing.assert_array_equal(p.global_ids[t][idx], parts[s].global_ids[t][a:b])
        # owned elements have no boundary face that is interior globally
        for t in p.types:
            for f in range(p.mesh.nbr[t].shape[1]):
                bl = p.mesh.nbr[t][:p.n_owned[t], f, 0] < 0
                gl = m.nbr[t][p.global_ids[t][:p.n_owned[t]], f, 0] < 0
                np.testing.assert_array_equal(bl, gl)
    assert total == {t: len(m.blocks[t]) for t in m.elem_types}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from layout_model import rhs as model_rhs
    from paper_1507_02557_b200.device import pack_mesh
    from paper_1507_02557_b200.dg import Discretization
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = build_mesh("hybrid:3")
        set_random_materials(m, 4)
        d = Discretization(m, 2, "GL", device="cpu")
        rng = np.random.default_rng(1)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        parts = build_local_parts(m, partition_elements(m, world, "rcb", N=2))
        p = parts[rank]
        dl = Discretization(p.mesh, 2, "GL", device="cpu")
        # local state: owned rows from the global state, ghost rows via gloo
        loc = {t: np.zeros((dl.n_elems[t], 4, dl.ops[t].Np)) for t in dl.types}
        for t in dl.types:
            loc[t][:p.n_owned[t]] = st[t][p.global_ids[t][:p.n_owned[t]]]
        reqs = []
        for s, per_t in p.send.items():
            for t, idx in per_t.items():
                reqs.append(dist.isend(torch.as_tensor(loc[t][idx].copy()), s))
        bufs = []
        for s, per_t in p.recv.items():
            for t, (a, b) in per_t.items():
                buf = torch.empty((b - a, 4, dl.ops[t].Np), dtype=torch.float64)
                reqs.append(dist.irecv(buf, s))
                bufs.append((t, a, b, buf))
        for r in reqs:
            r.wait()
        for t, a, b, buf in bufs:
            loc[t][a:b] = buf.numpy()
        got = model_rhs(pack_mesh(dl), dl, loc)
        ref = oracle.compute_rhs(d, st)
        err = 0.0
        for t in dl.types:
            own = p.global_ids[t][:p.n_owned[t]]
            g, r_ = got[t][:p.n_owned[t]], ref[t][own]
            err = max(err, float(np.abs(g - r_).max() / max(np.abs(r_).max(), 1e-300)))
        q.put((rank, err))
    finally:
        dist.destroy_process_group()


def test_partitioned_rhs_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err in res:
        assert err < 1e-12, (rank, err)


def _transport_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    from types import SimpleNamespace
    from paper_1507_02557_b200.mesh import structured_hybrid_mesh
    from paper_1507_02557_b200.parallel import NCCLTransport, make_parts
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = structured_hybrid_mesh(3, nx=3 * world)
        p = make_parts(m, world, "xslab", N=1, ranks=[rank])[rank]
        Np = {"hex": 8, "wedge": 6, "pyramid": 5, "tet": 4}
        # state rows carry their global id, so the receiver can check provenance
        qd = {t: torch.zeros((len(p.global_ids[t]), 4, Np[t]), dtype=torch.float64)
              for t in p.types}
        for t in p.types:
            qd[t][:p.n_owned[t]] = torch.as_tensor(
                p.global_ids[t][:p.n_owned[t]], dtype=torch.float64)[:, None, None]
        sendbuf = {peer: {t: qd[t][torch.as_tensor(idx)].clone() for t, idx in per_t.items()}
                   for peer, per_t in p.send.items()}
        ps = SimpleNamespace(
            send_buffers=lambda: [(pe, sendbuf[pe][t]) for pe in sorted(sendbuf)
                                  for t in p.types if t in sendbuf[pe]],
            recv_buffers=lambda qq: [(pe, qq[t][a:b]) for pe in sorted(p.recv)
                                     for t in p.types if t in p.recv[pe]
                                     for a, b in [p.recv[pe][t]]])
        tr = NCCLTransport()
        tr.wait(tr.start(ps, qd))
        ok = True
        for t in p.types:
            ghosts = qd[t][p.n_owned[t]:, 0, 0].numpy()
            ok &= bool(np.array_equal(ghosts, p.global_ids[t][p.n_owned[t]:].astype(float)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_halo_transport_batch_p2p_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_transport_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _face_halo_worker(rank, world, port, q, method, form):
    """4-rank face-level halo over gloo: each rank gathers the shared-face
    values of its owned elements (face nodes / published traces, the offsets
    the GPU path uses), exchanges them with the batched-P2P transport,
    scatters them into zeroed ghost rows and evaluates its owned elements
    with the numpy kernel model; must equal the whole-mesh oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from types import SimpleNamespace
    from layout_model import own_traces, rhs as model_rhs
    from paper_1507_02557_b200.device import pack_mesh
    from paper_1507_02557_b200.dg import Discretization
    from paper_1507_02557_b200.parallel import NCCLTransport, face_halo_offsets, flat_face_offsets
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 2
        m = build_mesh("hybrid:4")
        set_random_materials(m, 6)
        d = Discretization(m, N, form, device="cpu")
        rng = np.random.default_rng(3)
        st = {t: rng.standard_normal((d.n_elems[t], 4, d.ops[t].Np)) for t in d.types}
        p = build_local_parts(m, partition_elements(m, world, method, N=N))[rank]
        dl = Discretization(p.mesh, N, form, device="cpu")
        pk = pack_mesh(dl)
        sem = form == "SEM"
        loc = {t: np.zeros((dl.n_elems[t], 4, dl.ops[t].Np)) for t in dl.types}
        for t in dl.types:
            loc[t][:p.n_owned[t]] = st[t][p.global_ids[t][:p.n_owned[t]]]
        tr = {t: np.ascontiguousarray(own_traces(pk, t, loc[t], N, sem)) for t in dl.types}
        for t in dl.types:
            tr[t][p.n_owned[t]:] = 0.0                   # ghosts: only what the halo brings
        src, row, local, kind = {}, {}, {}, {}
        for t in dl.types:
            local[t], kind[t] = face_halo_offsets(t, pk["types"][t]["dops"], N, sem)
            src[t] = loc[t] if kind[t] == "state" else tr[t]
            row[t] = src[t].shape[1] * src[t].shape[2]
        send, recv = {}, {}
        for peer, per_t in p.send_faces.items():
            for t, pr in per_t.items():
                off = flat_face_offsets(pr, local[t], row[t])
                flat, stride = src[t].reshape(-1), row[t] // 4
                send.setdefault(peer, {})[t] = torch.as_tensor(
                    np.concatenate([flat[off + c * stride] for c in range(4)]))
        for peer, per_t in p.recv_faces.items():
            for t, pr in per_t.items():
                recv.setdefault(peer, {})[t] = torch.empty(
                    4 * len(flat_face_offsets(pr, local[t], row[t])), dtype=torch.float64)
        ps = SimpleNamespace(
            send_buffers=lambda: [(pe, send[pe][t]) for pe in sorted(send)
                                  for t in dl.types if t in send[pe]],
            recv_buffers=lambda qq: [(pe, recv[pe][t]) for pe in sorted(recv)
                                     for t in dl.types if t in recv[pe]])
        T = NCCLTransport()
        T.wait(T.start(ps, None))
        for peer, per_t in p.recv_faces.items():
            for t, pr in per_t.items():
                off = flat_face_offsets(pr, local[t], row[t])
                flat, stride, buf = src[t].reshape(-1), row[t] // 4, recv[peer][t].numpy()
                n = len(off)
                for c in range(4):
                    flat[off + c * stride] = buf[c * n:(c + 1) * n]
        got = model_rhs(pk, dl, loc, traces={t: tr[t] for t in dl.types if kind[t] == "trace"})
        ref = oracle.compute_rhs(d, st)
        err = 0.0
        for t in dl.types:
            own = p.global_ids[t][:p.n_owned[t]]
            g, r_ = got[t][:p.n_owned[t]], ref[t][own]
            err = max(err, float(np.abs(g - r_).max() / max(np.abs(r_).max(), 1e-300)))
        halo = sum(b.numel() for per_t in recv.values() for b in per_t.values())
        full = sum((b - a) * 4 * dl.ops[t].Np for per_t in p.recv.values()
                   for t, (a, b) in per_t.items())
        q.put((rank, err, halo, full))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("method,form", [("rcb", "GL"), ("xslab", "SEM")])
def test_face_halo_gloo_four_ranks(method, form):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 1000 + (7 if method == "xslab" else 0)
    procs = [ctx.Process(target=_face_halo_worker, args=(r, 4, port, q, method, form))
             for r in range(4)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err, halo, full in res:
        assert err < 1e-12, (rank, err)
        assert halo < full, (rank, halo, full)      # faces, not whole element states
