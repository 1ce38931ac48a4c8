"""Graph soak (not part of the test suite): a seeded random collective program
captured once and replayed many times - flag values re-based every replay -
with fresh inputs and a sha256 check against the oracle every k-th replay.
usage: graph_soak.py N SEED NOPS REPLAYS CHECK_EVERY [STICKY]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import _workers  # noqa: E402
from tests.test_stress_gpu import expected_digest  # noqa: E402


def main():
    n, seed, nops, replays, every = (int(a) for a in sys.argv[1:6])
    sticky = len(sys.argv) > 6 and sys.argv[6] == "1"
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("gsoak")
    t0 = time.time()
    res = launch(_workers.graph_stress_worker, d,
                 args=(key, n, seed, nops, replays, "mps", 0, sticky, every), job_key=key,
                 timeout_s=3000, mode="mps")
    ops = _workers.stress_ops(n, seed, nops)
    bad = checked = 0
    for rep in range(0, replays, every):
        for i, o in enumerate(ops):
            o_r = dict(o, seed=o["seed"] + 100_000 * rep)
            for r in range(n):
                checked += 1
                if res[r]["digests"][rep][i] != expected_digest(o_r, n, r):
                    bad += 1
                    print("MISMATCH", rep, i, o, r, flush=True)
    print(f"graph soak n={n} seed={seed} ops={nops} replays={replays} sticky={sticky}: "
          f"{checked} results checked, {'OK' if not bad else f'{bad} mismatches'} "
          f"({time.time() - t0:.0f} s)", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
