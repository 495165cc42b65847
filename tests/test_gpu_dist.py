"""The multi-process training path on the GPU: one process per shard
(DGNNTrainer(distributed=True) -> NcclRunner), here 2 ranks sharing cuda:0
over the gloo backend, D = 2 and 4 (the round's box has one GPU; the runner code is
backend-agnostic: MAX/SUM all-reduce, variable-count all_to_all_single),
against the single-process LocalRunner on the same reference plans
with adaptive staleness on: identical losses, stale decisions and parameters."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

EPOCHS = 3


def _cfg():
    from paper_2309_03523_b200 import DGNNConfig
    return DGNNConfig(F=16, H=16, C=16, rnn="lstm", n_rnn=2, optimizer="adam", lr=1e-2,
                      precision="fp32")


def _run(distributed, plan="t2", stale="relax"):
    from pathlib import Path
    from paper_2309_03523_b200 import StaleConfig, load_plan_npz
    from paper_2309_03523_b200.model import init_params, synthetic_inputs
    from paper_2309_03523_b200.trainer import DGNNTrainer
    pa = load_plan_npz(Path(__file__).resolve().parents[1] / "artifacts" / plan / "plan.npz")
    cfg = _cfg()
    X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
    scfg = StaleConfig.adaptive() if stale == "relax" else StaleConfig.off()
    tr = DGNNTrainer(pa, cfg, scfg, features=X, labels=y,
                     params=init_params(cfg, 0), device="cuda:0", distributed=distributed)
    reps = [tr.run_epoch() for _ in range(EPOCHS)]
    sends = [{k: c.send.cpu().numpy().copy() for k, c in
              [(f"s{l}", sh.scache[l]) for l in range(2)] + [(f"t{k}", sh.tcache[k]) for k in range(cfg.n_rnn)]}
             if sh.stale_on else {} for sh in tr.shards]
    return ([r.loss for r in reps], [r.stale_sent_bytes for r in reps], tr.params(0), sends)


def _worker(rank, world, plan, stale, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(True, plan, stale)))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("plan,world,stale,port", [("t2", 2, "relax", 29571), ("t4", 4, "relax", 29572),
                                                   ("t2", 2, "off", 29573), ("t4", 4, "off", 29574)])
def test_distributed_runner_equals_local_runner(plan, world, stale, port):
    """stale "off" exercises the static-count exchanges (no count all-to-all)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, plan, stale, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(got[r], str), got[r]
    loss_l, sent_l, params_l, sends_l = _run(False, plan, stale)
    # 2 ranks: every all-reduce sums 2 operands (exact, order-free) -> bitwise
    # equal. 4 ranks: gloo's gradient SUM order differs from the local runner's
    # sequential order, so later epochs differ by float rounding (~1e-10)
    exact = world == 2
    for r in range(world):
        loss_d, sent_d, params_d, sends_d = got[r]
        assert loss_d[0] == loss_l[0]
        if exact:
            assert loss_d == loss_l, (r, loss_d, loss_l)
        else:
            np.testing.assert_allclose(loss_d, loss_l, rtol=1e-6)
        assert sent_d == sent_l
        for k in params_l:
            if exact:
                np.testing.assert_array_equal(params_d[k], params_l[k], err_msg=k)
            else:
                np.testing.assert_allclose(params_d[k], params_l[k], rtol=1e-5, atol=1e-7, err_msg=k)
        for k in sends_d[0]:
            np.testing.assert_array_equal(sends_d[0][k], sends_l[r][k], err_msg=k)
