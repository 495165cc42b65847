"""The N>1 host logic on CPU: the NCCL runner (here over gloo, world size 2
and 3) delivers exactly what the single-process LocalRunner delivers for the
same generator protocol (MAX all-reduce, variable-count all-to-allv with
empty peers, SUM all-reduce), and per-rank layouts agree on every exchange."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def mock_step(d, D):
    """Mimics Shard.step's collective protocol on CPU tensors."""
    out = {}
    m = yield ("max", torch.tensor([float(d * 3 % 5)]))
    out["max"] = float(m.item())
    peers = [p for p in range(D) if p != d]
    bufs, idxs = [], []
    for p in peers:
        c = (d * 7 + p * 3) % 5  # includes empty sends
        bufs.append(torch.arange(c * 4, dtype=torch.float32).view(c, 4) + 100 * d + 10 * p)
        idxs.append(torch.arange(c, dtype=torch.int32) * 2 + d)
    rb, ri = yield ("a2av", bufs, idxs)
    out["recv"] = {p: (b.clone().numpy(), i.clone().numpy()) for p, b, i in zip(peers, rb, ri)}
    # second exchange with different widths (the temporal carry path: 2H wide)
    bufs2 = [torch.full((1, 8), float(d * 10 + p)) for p in peers]
    idx2 = [torch.tensor([p], dtype=torch.int32) for p in peers]
    rb2, ri2 = yield ("a2av", bufs2, idx2)
    out["recv2"] = {p: (b.clone().numpy(), i.clone().numpy()) for p, b, i in zip(peers, rb2, ri2)}
    g = torch.full((6,), float(d + 1))
    s = yield ("sum", g)
    out["sum"] = s.clone().numpy()
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2309_03523_b200.trainer import NcclRunner
    (res,) = NcclRunner().run([mock_step(rank, world)])
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,port", [(2, 29561), (3, 29562)])
def test_nccl_runner_equals_local_runner(world, port):
    from paper_2309_03523_b200.trainer import LocalRunner
    local = LocalRunner().run([mock_step(d, world) for d in range(world)])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for d in range(world):
        a, b = local[d], got[d]
        assert a["max"] == b["max"] == max(float(r * 3 % 5) for r in range(world))
        np.testing.assert_array_equal(a["sum"], b["sum"])
        for key in ("recv", "recv2"):
            for p in a[key]:
                np.testing.assert_array_equal(a[key][p][0], b[key][p][0])
                np.testing.assert_array_equal(a[key][p][1], b[key][p][1])
                # sender p's payload for d arrives intact
                if key == "recv":
                    c = (p * 7 + d * 3) % 5
                    assert a[key][p][0].shape == (c, 4)


@pytest.mark.parametrize("name", ["t2", "t4", "c1"])
def test_rank_layouts_agree_on_exchanges(artifacts_dir, name):
    from paper_2309_03523_b200 import load_plan_npz
    from paper_2309_03523_b200.layout import build_layout
    pa = load_plan_npz(artifacts_dir / name / "plan.npz")
    lays = [build_layout(pa, d) for d in range(pa.n_devices)]
    succ = np.full(pa.n_instances, -1)
    succ[pa.temporal_links[:, 0]] = pa.temporal_links[:, 1]
    for d, ld in enumerate(lays):
        for p, lp in enumerate(lays):
            if p == d:
                continue
            sp = ld.send_pos[ld.send_ptr[p]:ld.send_ptr[p + 1]]
            sent_gid = ld.own_gid[ld.key_rows[sp]]
            rs = lp.recv_slot[lp.recv_ptr[d]:lp.recv_ptr[d + 1]]
            recv_gid = lp.halo_gid[rs - lp.n_own]
            np.testing.assert_array_equal(sent_gid, recv_gid)
            tp = ld.tsend_pos[ld.tsend_ptr[p]:ld.tsend_ptr[p + 1]]
            tsent = ld.own_gid[ld.tkey_rows[tp]]
            carries = lp.trecv_carry[lp.trecv_ptr[d]:lp.trecv_ptr[d + 1]]
            run_of_carry = {int(c): r for r, c in enumerate(lp.run_carry) if c >= 0}
            preds = np.asarray([lp.run_pred_gid[run_of_carry[int(c)]] for c in carries])
            np.testing.assert_array_equal(tsent, preds)
            # the successor of every carried predecessor is the first row of its run
            firsts = [lp.own_gid[lp.run_rows[lp.run_ptr[run_of_carry[int(c)]]]] for c in carries]
            np.testing.assert_array_equal(succ[tsent], firsts)
