"""Multi-process (torch.distributed gloo, world_size 2) checks of the executor's rank logic.

Every rank asks libgx.so for its own device-free topology (gx_exec_topology, "dryrun" comm):
communication group member lists, per-layer data chunks and pipeline send/recv lists.  The
views are exchanged with all_gather_object and cross-checked — exactly the agreements the
NCCL path relies on (identical group pool on every rank, every send matched by one receive
of the same sample range, chunks partitioning each micro-batch).  World sizes up to 8 are
covered by giving each of the 2 processes half of the ranks.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_13878_b200 import executor as gxe

PLANS = [
    # (world, strategies, batch, pp, micro_batches)
    (2, ["dp:2", "sdp:2", "tp:2", "dp:2"], 4, 1, 1),
    (4, ["tp:2,sdp:2", "dp:4", "tp:4", "sdp:4"], 6, 1, 1),
    (8, ["tp:2,dp:2", "sdp:4", "dp:2,tp:2", "tp:4"], 8, 2, 2),
    (8, ["dp:2", "tp:2", "sdp:2", "dp:2", "tp:2", "tp:2", "sdp:2", "dp:2"], 8, 4, 4),
    (8, ["", "", "", "", "", "", "", ""], 8, 8, 8),
    (8, ["sdp:8", "dp:8", "tp:8", "tp:2,sdp:4"], 17, 1, 1),
]


def _model(L):
    shape = {"hidden": 256, "heads": 8, "head_dim": 32, "seq": 16, "ffn": 512, "kind": "encoder"}
    return {"dtype_bytes": 4, "layers": [{"param_bytes": 1, "activation_bytes_per_sample": 1,
                                          "fwd_time_per_sample_ms": 0.1, "shape": dict(shape)}
                                         for _ in range(L)]}


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for (N, strategies, B, pp, m) in PLANS:
        plan = gxe.make_plan(strategies, B, pp, m)
        mine = [r for r in range(N) if r % world == rank]
        topo = gxe.topology(plan, _model(len(strategies)), N, mine)
        views = [None] * world
        dist.all_gather_object(views, topo)
        out.append(views)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def gathered():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("i", range(len(PLANS)))
def test_rank_views_agree(gathered, i):
    N, strategies, B, pp, m = PLANS[i]
    views = gathered[i]
    # identical group pool (registration order) on every process
    assert all(v["groups"] == views[0]["groups"] for v in views)
    ranks = {r["rank"]: r for v in views for r in v["ranks"]}
    assert sorted(ranks) == list(range(N))
    g = N // pp
    Bm = B // m
    for r in ranks.values():
        for L in r["layers"]:
            for key in ("tp_group", "sdp_group", "dp_group", "relayout_group"):
                members = L[key]
                if members is None:
                    continue
                assert r["rank"] in members
                for other in members:  # every member sees the same group
                    OL = next(x for x in ranks[other]["layers"] if x["layer"] == L["layer"])
                    assert OL[key] == members
    # data chunks: TP replicas share a chunk; the D chunks partition every micro-batch
    for st in range(pp):
        stage_ranks = [ranks[st * g + i] for i in range(g)]
        for li in range(len(stage_ranks[0]["layers"])):
            for mb in range(m):
                chunks = {}
                for r in stage_ranks:
                    L = r["layers"][li]
                    chunks.setdefault(L["data_rank"], set()).add(tuple(L["chunks"][mb]))
                assert all(len(c) == 1 for c in chunks.values())
                spans = sorted(next(iter(c)) for c in chunks.values())
                assert spans[0][0] == mb * Bm and spans[-1][1] == (mb + 1) * Bm
                assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    # pipeline: every send has exactly one matching receive (same micro-batch and range)
    for fwd_send, recv in ((0, 1), (2, 3)):
        sends = [(r["rank"], x["peer"], x["mb"], x["lo"], x["hi"]) for r in ranks.values()
                 for x in r["pp"] if x["kind"] == fwd_send]
        recvs = [(x["peer"], r["rank"], x["mb"], x["lo"], x["hi"]) for r in ranks.values()
                 for x in r["pp"] if x["kind"] == recv]
        assert sorted(sends) == sorted(recvs)
        # each receiver's pieces tile its own chunk
        for r in ranks.values():
            for mb in range(m):
                pieces = sorted((x["lo"], x["hi"]) for x in r["pp"] if x["kind"] == recv and x["mb"] == mb)
                if not pieces:
                    continue
                assert all(a[1] == b[0] for a, b in zip(pieces, pieces[1:]))
