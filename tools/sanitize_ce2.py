"""Two ranks on one GPU, copy-engine transport, multi-round pipeline: the
two-ranks-per-GPU schedule (fetch on the gather lane into a double-buffered
scratch; with FMX_RCE_ROUNDS=1 the result slot by copy engine every round),
checked against the oracle - small enough to run under compute-sanitizer
(memcheck / synccheck, FMX_SERIALIZE=1, --target-processes all).

usage: python tools/sanitize_ce2.py [count]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rank_main(rank: int, job_key: str, count: int):
    import torch

    from oracle import oracle as orc
    from paper_2511_09143_b200 import instance
    from paper_2511_09143_b200.comm import init_process_group

    inst = instance.bind(0, rank + 1, mode="green")
    # 64 KiB slices: a few MB span many rounds
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=2, transport="ce",
                              slice_bytes=64 << 10, timeout_s=120)
    s = inst.stream
    x = orc.synthetic_gradient(rank, count, orc.F32)
    with torch.cuda.stream(s):
        t = torch.from_numpy(x).to("cuda")
    s.synchronize()
    for _ in range(2):
        comm.allreduce(t, op="avg", stream=s)
        with torch.cuda.stream(s):
            t.copy_(torch.from_numpy(x).to("cuda"))
    comm.allreduce(t, op="avg", stream=s)
    s.synchronize()
    out = t.cpu().numpy()
    comm.destroy()
    return out


if __name__ == "__main__":
    from oracle import oracle as orc
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    count = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_003
    want = orc.allreduce_c([orc.synthetic_gradient(r, count, orc.F32) for r in range(2)],
                           orc.F32, *orc.ddp_mean(2))
    d = fm_select(Job(0, "train", 2, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("san")
    res = launch(rank_main, d, args=(key, count), job_key=key, mode="green", timeout_s=900,
                 inline_rank0=True)
    for r, out in enumerate(res):
        assert np.array_equal(out.view(np.uint32), want.view(np.uint32)), f"rank {r} mismatch"
    print(f"ok: 2 ranks, {count} f32, copy-engine pipeline with the fetch lane, bit-exact")
