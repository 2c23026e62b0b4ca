"""Times the distributed four-step NDCT / NDCT^T against the single-GPU
multi-pass NDCT stage at one N on one B200 (world 1: the exchange is the
identity; with P emulated ranks, each rank's local work one after another
to show the per-rank cost). Usage: python tools/time_four_step.py [log2n] [world]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import distributed as D  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = []
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        b.synchronize()
        best.append(a.elapsed_time(b))
    return min(best), sorted(best)[len(best) // 2]


def main():
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    n = 1 << log2n
    cfg = fl.TransformConfig(n)
    terms = D.stage_terms(cfg, D.STAGE_NDCT)
    c = torch.from_numpy(fl.random_decaying(n, 1.0, 3)).cuda()
    out = torch.empty_like(c)
    print("multi-pass NDCT     ms", timed(lambda: D.gpu_stage(cfg, 0, D.STAGE_NDCT, 0, terms, c, out)))
    print("multi-pass NDCT^T   ms", timed(lambda: D.gpu_stage(cfg, 1, D.STAGE_NDCT, 0, terms, c, out)))
    fs = D.FourStep(cfg, 1, 0)
    comm = D.TorchComm(None)
    chat = fs.to_residue(c)
    for groups in (fs.groups(), fs.groups(min_groups=2), [(t, t + 1) for t in range(terms)]):
        print("four-step NDCT      ms", len(groups), "groups",
              timed(lambda: D._ndct_four_step(fs, comm, chat, groups)))
        print("four-step NDCT^T    ms", len(groups), "groups",
              timed(lambda: D._ndct_t_four_step(fs, comm, c, groups)))
    print("to_residue          ms", timed(lambda: fs.to_residue(c)))
    print("whole dlt_four_step ms", timed(lambda: D.dlt_four_step(cfg, c, None, fs), 3))
    print("whole D.dlt         ms", timed(lambda: D.dlt(cfg, c), 3))
    print("whole idlt_four_step ms", timed(lambda: D.idlt_four_step(cfg, c, None, fs), 3))
    print("whole D.idlt        ms", timed(lambda: D.idlt(cfg, c), 3))


if __name__ == "__main__":
    main()
