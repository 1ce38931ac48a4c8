"""Generate tests/golden/allreduce_golden.npz: small allreduce vectors whose
expected outputs are computed with TORCH (fp32 elementwise adds in ascending
rank order, torch.div / torch.mul for the scale conventions, torch's bf16
conversion for rounding) - an implementation independent of oracle/.

The reference has no allreduce arithmetic to generate these from (its data
path is NCCL), so these pin the oracle to the contract as
torch evaluates it, not to the reference."""

import os

import numpy as np
import torch

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "allreduce_golden.npz")


def torch_allreduce(xs, dtype, op, factor):
    ts = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).float() if dtype == 1
          else torch.from_numpy(x) for x in xs]
    if op == 2:
        ts = [t / torch.tensor(factor, dtype=torch.float32) for t in ts]
        if dtype == 1:
            ts = [t.to(torch.bfloat16).float() for t in ts]
    acc = ts[0].clone()
    for t in ts[1:]:
        acc = acc + t
    if op == 1:
        acc = acc * torch.tensor(factor, dtype=torch.float32)
    if dtype == 1:
        return acc.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    return acc.numpy()


def main():
    rng = np.random.default_rng(2511)
    arrays = {}
    cases = [(2, 0, 0, 1.0), (3, 0, 1, 0.5), (7, 0, 2, 7.0), (7, 1, 0, 1.0), (7, 1, 2, 7.0),
             (4, 1, 1, 0.25), (14, 0, 2, 14.0)]
    for i, (n, dtype, op, factor) in enumerate(cases):
        count = int(rng.integers(1, 300))
        xs = []
        for r in range(n):
            x = (rng.standard_normal(count) * 10 ** rng.uniform(-6, 6)).astype(np.float32)
            x[rng.random(count) < 0.05] = np.float32(1e8) * (1 if r % 2 else -1)
            if dtype == 1:
                x = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
            xs.append(x)
        stem = f"case{i}"
        for r, x in enumerate(xs):
            arrays[f"{stem}_in{r}"] = x
        arrays[f"{stem}_meta"] = np.array([n, dtype, op, factor], dtype=np.float64)
        arrays[f"{stem}_out"] = torch_allreduce(xs, dtype, op, factor)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
