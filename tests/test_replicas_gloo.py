"""Multi-process replica sharding on CPU (gloo, world_size 2): the N>1 host logic of
SURVEY §8(e) R.  Each rank counts its colourings with the CPU oracle (test
infrastructure) and the all-reduce must reproduce the single-process vector and
estimate exactly, in U64 and F64."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2009_11665_b200.replicas import count_replicated, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_every_colouring_once():
    for n in range(0, 23):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                first, stride, cnt = shard(n, r, world, iter_offset=5)
                seen += [first + stride * t for t in range(cnt)]
            assert sorted(seen) == list(range(5, 5 + n))


def test_vertex_partition_rows_tile_the_graph():
    # contiguous row blocks, disjoint, covering [0, n) in rank order,
    # at most ceil(n / world) rows each (n < world and n = 0 leave empty ranks)
    from paper_2009_11665_b200.sg2v import partition_rows
    for n in (0, 1, 2, 7, 8, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            nxt = 0
            for r in range(world):
                b, nl = partition_rows(n, r, world)
                assert nl >= 0 and nl <= -(-n // world)
                assert b == nxt or nl == 0
                nxt = b + nl if nl else nxt
            assert nxt == n


def _oracle_count_fn(case):
    from oracle import oracle as O

    def fn(g, t, n, seed, prec, off, stride):
        arith = O.ARITH_U64 if prec == "u64" else O.ARITH_F64
        out = []
        for q in range(n):
            j = off + q * stride
            r = O.count(case["g"], case["k"], case["e"], O.colors(seed, j, case["g"].n, case["k"]), arith=arith)
            out.append(r if prec == "u64" else r[0])
        return np.array(out, dtype=np.uint64 if prec == "u64" else np.float64)
    return fn


def _case():
    from sg2v_inputs import erdos_renyi, TEMPLATES
    from oracle import oracle as O
    import paper_2009_11665_b200 as sg
    e = TEMPLATES["u5-2"]
    # the library's template handle (host-only): a7 runs in the C ABI (sg2v_estimate)
    return {"g": erdos_renyi(200, 900, seed=3), "k": 5, "e": e, "info": sg.template_build(5, e),
            "P": float(O.colorful_probability(5)), "alpha": O.alpha(5, e)}


def _worker(rank, world, port, n_iter, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = _case()
    res = {}
    for prec in ("u64", "f64"):
        est, full = count_replicated(case["g"], case["info"], n_iter, seed=9, precision=prec, rank=rank,
                                     world=world, count_fn=_oracle_count_fn(case))
        res[prec] = (est, full.tolist())
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, res))


@pytest.mark.parametrize("n_iter", [7, 8])
def test_gloo_world2_matches_single_process(n_iter):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_iter, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = _case()
    for prec in ("u64", "f64"):
        est1, full1 = count_replicated(case["g"], case["info"], n_iter, seed=9, precision=prec,
                                       count_fn=_oracle_count_fn(case))
        for r in (0, 1):
            est, full = out[r][prec]
            assert full == full1.tolist()
            if prec == "u64":
                assert math.isnan(est)
            else:
                assert est == est1
                assert math.isclose(est, sum(full1) / n_iter / (case["P"] * case["alpha"]), rel_tol=1e-12)
