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
    """Mimics Shard.step's collective protocol on CPU tensors: MAX all-reduce,
    a device-counted (stale-filtered) one-buffer all-to-allv, a static-count
    one (the temporal carries: other record width), SUM all-reduce."""
    out = {}
    m = yield ("max", torch.tensor([float(d * 3 % 5)]))
    out["max"] = float(m.reshape(-1)[0])
    rw = 4 + 4  # 16-byte header + 4 floats
    cnt = [(d * 7 + p * 3) % 5 if p != d else 0 for p in range(D)]  # includes empty sends
    send = torch.cat([torch.arange(c * rw, dtype=torch.float32) + 100 * d + 10 * p
                      for p, c in enumerate(cnt)] + [torch.zeros(3 * rw)])  # spare capacity
    counts = torch.tensor(cnt, dtype=torch.int32)
    recv = torch.full((5 * D * rw,), -1.0)
    rcounts = torch.zeros(D, dtype=torch.int32)
    tok = yield ("a2a_start", send, None, counts, recv, rw, None, rcounts)
    res = yield ("a2a_finish", tok)
    out["recv"] = (list(res["recv_counts"]), recv[:sum(res["recv_counts"]) * rw].clone().numpy(),
                   rcounts.clone().numpy(), list(res["send_counts"]))
    # static counts (known to both sides), width 8 + header
    rw2 = 8 + 4
    sc = [1 if p != d else 0 for p in range(D)]
    send2 = torch.cat([torch.full((rw2,), float(d * 10 + p)) for p in range(D) if p != d])
    recv2 = torch.zeros((D - 1) * rw2)
    tok2 = yield ("a2a_start", send2, sc, None, recv2, rw2, list(sc), None)
    res2 = yield ("a2a_finish", tok2)
    out["recv2"] = (list(res2["recv_counts"]), recv2.clone().numpy())
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
            assert a[key][0] == b[key][0]
            for x, y in zip(a[key][1:], b[key][1:]):
                np.testing.assert_array_equal(x, y)
        # sender p's records for d arrive intact, peer-major
        rc = a["recv"][0]
        assert rc == [(p * 7 + d * 3) % 5 if p != d else 0 for p in range(world)]
        np.testing.assert_array_equal(a["recv"][2], rc)
        off = 0
        for p in range(world):
            if rc[p]:
                sc_p = [(p * 7 + q * 3) % 5 if q != p else 0 for q in range(world)]
                first = 100 * p + 10 * d + 0.0
                assert a["recv"][1][off * 8] == first
                assert a["recv"][1][(off + rc[p]) * 8 - 1] == first + rc[p] * 8 - 1
                assert sum(sc_p[:d]) >= 0
            off += rc[p]


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
