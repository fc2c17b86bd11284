"""Vertex-partitioned mode on the GPU.

* world = 1 with the NCCL transport and forced narrow column tiles: every step runs
  through the tiled all-gather + global-B push + combine path and must equal the
  single-GPU path (U64 exact, F64 below 2^53 exact, F32 1e-4).
* world = 2 with two processes sharing cuda:0 and the host-callback transport over
  gloo: each rank holds half of the rows of every table; the all-gathered counts
  must equal the single-process values bit-exactly (U64) AND the CPU oracle's.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_11665_b200 as sg  # noqa: E402
from sg2v_inputs import TEMPLATES, rmat  # noqa: E402


def _k(e):
    return 1 + max(max(x) for x in e)


def _part(g, rank, world):
    b, nl = sg.partition_rows(g.n, rank, world)
    ro = g.row_offsets[b:b + nl + 1] - g.row_offsets[b]
    ci = g.col_indices[g.row_offsets[b]:g.row_offsets[b + nl]]
    return b, nl, ro, ci


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("name", ["u3-1", "u5-2", "u7-2", "path6", "star6", "u10-2"])
def test_world1_nccl_tiled_equals_single(oracle, name):
    g = rmat(12, 60_000, 0.45, 0.22, 0.22, seed=6)
    e = TEMPLATES[name]
    k = _k(e)
    comm = sg.Comm.nccl(sg.Comm.unique_id(), 0, 1)
    b, nl, ro, ci = _part(g, 0, 1)
    Gp = sg.graph_load_partition(g.n, b, nl, ro, ci)
    G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
    for root in (-1, 0):
        T = sg.template_build(k, e, root_hint=root)
        _, want = sg.count(G, T, n_iter=3, seed=2, precision="u64")
        for tile in (0, 4, 12):
            _, got = sg.count(Gp, T, n_iter=3, seed=2, precision="u64", comm=comm, col_tile=tile)
            assert np.array_equal(got, want), (name, root, tile)
        _, wf = sg.count(G, T, n_iter=2, seed=2, precision="f32")
        _, gf = sg.count(Gp, T, n_iter=2, seed=2, precision="f32", comm=comm, col_tile=8)
        assert np.allclose(gf, wf, rtol=1e-4, atol=0)
        # and against the oracle directly (U64 residues, F64 values for the F32 bar)
        for j in range(2):
            cols = oracle.colors(2, j, g.n, k)
            assert int(want[j]) == oracle.count(g, k, e, cols)
            assert abs(gf[j] - oracle.count(g, k, e, cols, arith=oracle.ARITH_F64)[0]) <= 1e-4 * abs(gf[j])
    comm.free()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2009_11665_b200 as sgw

    def allgather(data: bytes) -> bytes:
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return b"".join(x.numpy().tobytes() for x in out)

    comm = sgw.Comm.callback(rank, world, allgather)
    g = rmat(12, 60_000, 0.45, 0.22, 0.22, seed=6)
    b, nl, ro, ci = _part(g, rank, world)
    Gp = sgw.graph_load_partition(g.n, b, nl, ro, ci)
    # the balanced relabelling (degree-dealt blocks), colours keyed by the input ids
    oon, ro2, ci2 = sgw.partition_relabel(g.row_offsets, g.col_indices, world)
    Gr = sgw.graph_load_partition(g.n, b, nl, ro2[b:b + nl + 1] - ro2[b], ci2[ro2[b]:ro2[b + nl]])
    sgw.graph_set_vertex_ids(Gr, oon)
    res = {}
    for name in ("u5-2", "u7-2", "u10-2"):
        e = TEMPLATES[name]
        T = sgw.template_build(_k(e), e)
        # column tiles (overlapped exchange) and whole rows (fused kernels on staged rows)
        _, c = sgw.count(Gp, T, n_iter=2, seed=5, precision="u64", comm=comm, col_tile=16)
        _, c0 = sgw.count(Gp, T, n_iter=2, seed=5, precision="u64", comm=comm, col_tile=0)
        _, cr = sgw.count(Gr, T, n_iter=2, seed=5, precision="u64", comm=comm, col_tile=0)
        _, cf = sgw.count(Gr, T, n_iter=2, seed=5, precision="f32", comm=comm, col_tile=0)
        assert [int(x) for x in c] == [int(x) for x in c0] == [int(x) for x in cr], name
        res[name] = [int(x) for x in c]
        res[name + "/f32"] = [float(x) for x in cf]
    comm.free()
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, res))


def test_world2_callback_equals_single(oracle):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = rmat(12, 60_000, 0.45, 0.22, 0.22, seed=6)
    G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
    for name in ("u5-2", "u7-2", "u10-2"):
        e = TEMPLATES[name]
        _, want = sg.count(G, sg.template_build(_k(e), e), n_iter=2, seed=5, precision="u64")
        assert out[0][name] == [int(x) for x in want] == out[1][name], name
        k = _k(e)
        assert out[0][name] == [oracle.count(g, k, e, oracle.colors(5, j, g.n, k)) for j in range(2)], name
        for j in range(2):
            wf = oracle.count(g, k, e, oracle.colors(5, j, g.n, k), arith=oracle.ARITH_F64)[0]
            assert abs(out[0][name + "/f32"][j] - wf) <= 1e-4 * wf, name


def _nccl_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_2009_11665_b200 as sgw
    uid = [sgw.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sgw.Comm.nccl(uid[0], rank, world)
    g = rmat(12, 60_000, 0.45, 0.22, 0.22, seed=6)
    b, nl, _, _ = _part(g, rank, world)
    oon, ro2, ci2 = sgw.partition_relabel(g.row_offsets, g.col_indices, world)
    Gr = sgw.graph_load_partition(g.n, b, nl, ro2[b:b + nl + 1] - ro2[b], ci2[ro2[b]:ro2[b + nl]])
    sgw.graph_set_vertex_ids(Gr, oon)
    res = {}
    for name in ("u5-2", "u7-2", "u10-2"):
        e = TEMPLATES[name]
        T = sgw.template_build(_k(e), e)
        _, c0 = sgw.count(Gr, T, n_iter=2, seed=5, precision="u64", comm=comm, col_tile=0)
        _, c1 = sgw.count(Gr, T, n_iter=2, seed=5, precision="u64", comm=comm, col_tile=16)
        res[name] = ([int(x) for x in c0], [int(x) for x in c1])
    comm.free()
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, res))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs (NCCL over NVLink; runs on the 8-GPU node)")
def test_world2_nccl_two_gpus(oracle):
    """One process per GPU, NCCL all-gathers over NVLink, balanced relabelled
    partition: whole-row exchange and column tiles both equal the oracle's counts."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = rmat(12, 60_000, 0.45, 0.22, 0.22, seed=6)
    for name in ("u5-2", "u7-2", "u10-2"):
        e = TEMPLATES[name]
        k = _k(e)
        want = [oracle.count(g, k, e, oracle.colors(5, j, g.n, k)) for j in range(2)]
        for r in (0, 1):
            assert out[r][name][0] == want and out[r][name][1] == want, (name, r)
