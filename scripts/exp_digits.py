"""How many e4m3 digits of Zq does the 1e-3 budget need?  (host-only numerics study, numpy)

Emulates the decode's operand format on the synthetic recipe (synthetic.make_random_blocks,
channel gains with outliers): per block i and 128-column unit, Z = V'_i (x / s) is scaled by
2^e_u (largest |Z| of the unit <= 448) and split greedily into e4m3 digits d0 + d1 + d2 (round to
nearest even, subnormals down to 2^-9); the sign contraction and the U' epilogue are exact.
Prints the relative L2 error of y = W_hat_n x against fp64 for 1, 2 and 3 digits.
Usage: python scripts/exp_digits.py [d_out_sample d_in n]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from synthetic import make_random_blocks, make_x  # noqa: E402
from synthetic.generators import channel_gains  # noqa: E402


def e4m3(v):
    a = np.abs(v)
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    e = np.maximum(e, -6.0)
    q = np.exp2(e - 3)
    r = np.minimum(np.round(a / q) * q, 448.0)
    return np.where(a > 0, np.sign(v) * r, 0.0)


def main(d_out=256, d_in=4096, n=4, k=16, seeds=(1, 2, 3)):
    for seed in seeds:
        signs, u, v, s = make_random_blocks(n, d_out, d_in, k, seed=seed)
        x = make_x(1, channel_gains(d_in, seed + 1), seed + 7)[0]
        bits = np.unpackbits(signs, axis=1, bitorder="little")[:, : d_out * d_in].reshape(n, d_out, d_in)
        S = bits.astype(np.float64) * 2 - 1
        xs = x / s.astype(np.float64)
        y = np.zeros(d_out)
        yq = {1: np.zeros(d_out), 2: np.zeros(d_out), 3: np.zeros(d_out)}
        for i in range(n):
            Z = v[i].astype(np.float64) * xs[:, None]                     # [d_in, k]
            y += np.einsum("or,or->o", u[i], S[i] @ Z)
            Zd = {1: np.zeros_like(Z), 2: np.zeros_like(Z), 3: np.zeros_like(Z)}
            for c0 in range(0, d_in, 128):
                blk = Z[c0:c0 + 128]
                m = np.abs(blk).max()
                if m == 0:
                    continue
                e_u = np.floor(np.log2(448.0 / m))
                if m * 2.0 ** e_u > 448.0:
                    e_u -= 1
                zz = blk * 2.0 ** e_u
                d0 = e4m3(zz)
                d1 = e4m3(zz - d0)
                d2 = e4m3(zz - d0 - d1)
                Zd[1][c0:c0 + 128] = d0 / 2.0 ** e_u
                Zd[2][c0:c0 + 128] = (d0 + d1) / 2.0 ** e_u
                Zd[3][c0:c0 + 128] = (d0 + d1 + d2) / 2.0 ** e_u
            for nd in (1, 2, 3):
                yq[nd] += np.einsum("or,or->o", u[i], S[i] @ Zd[nd])
        errs = {nd: np.linalg.norm(yq[nd] - y) / np.linalg.norm(y) for nd in (1, 2, 3)}
        print(f"seed {seed}: d_out {d_out} d_in {d_in} n {n}: rel L2  1 digit {errs[1]:.2e}  "
              f"2 digits {errs[2]:.2e}  3 digits {errs[3]:.2e}")


if __name__ == "__main__":
    a = [int(t) for t in sys.argv[1:4]]
    main(*a) if a else main()
