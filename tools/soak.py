"""Extended soak (not part of the test suite): seeded random collective programs,
sha256-exact against the oracle.  usage: soak.py N GPUS MODE SEED NOPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import _workers  # noqa: E402
from tests.test_stress_gpu import expected_digest  # noqa: E402


def main():
    n, gpus, mode, seed, nops = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job
    if gpus > 1:
        os.environ["FMX_FAKE_BUS"] = "1"
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", gpus))
    key = new_job_key("soak")
    res = launch(_workers.stress_worker, d, args=(key, n, seed, nops, mode), job_key=key,
                 timeout_s=3000, mode=mode, gpu_map={g: "0" for g in range(gpus)})
    ops = _workers.stress_ops(n, seed, nops)
    bad = 0
    for i, o in enumerate(ops):
        for r in range(n):
            if res[r]["digests"][i] != expected_digest(o, n, r):
                bad += 1
                print("MISMATCH", i, o, r, flush=True)
    print(f"soak n={n} gpus={gpus} mode={mode} seed={seed} ops={nops}: {'OK' if not bad else f'{bad} mismatches'}",
          flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
