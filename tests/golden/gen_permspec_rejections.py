"""Writes tests/golden/permspec_v1_rejections.txt: PERM-SPEC v1 group-1 sets for
permutations in which Lemire's bounded draw REJECTS at least one main-stream word, so the
side-stream branch (counter (q', b, s, 1 + i), words taken in order) decides the set.

Independent of oracle/ and of the CUDA library: Philox4x32-10 is written here from the
Salmon et al. (SC'11) round definition (checked below against the Random123 known-answer
vector of tests/golden/philox_kat.txt before anything is written), and the shuffle is a
SPARSE partial Fisher-Yates (a dict of displaced positions instead of an N-element array),
i.e. a different realisation of DESIGN.md R6 than the oracle's array swap.

    python tests/golden/gen_permspec_rejections.py   (about a minute of pure Python)
"""
from __future__ import annotations

import hashlib
import os

M0, M1 = 0xD2511F53, 0xCD9E8D57          # Philox multipliers
W0, W1 = 0x9E3779B9, 0xBB67AE85          # Weyl key increments
MASK = 0xFFFFFFFF


def philox(ctr, key):
    x0, x1, x2, x3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0, p1 = M0 * x0, M1 * x2
        x0, x1, x2, x3 = ((p1 >> 32) ^ x1 ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ x3 ^ k1) & MASK, p0 & MASK
        k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return (x0, x1, x2, x3)


class Stream:
    """Words w_0, w_1, ... of the stream with counter words (c1, c2, c3)."""

    def __init__(self, key, c1, c2, c3):
        self.key, self.c = key, (c1, c2, c3)
        self.q, self.buf = -1, None

    def word(self, idx):
        q = idx // 4
        if q != self.q:
            self.q, self.buf = q, philox((q,) + self.c, self.key)
        return self.buf[idx % 4]


def group1(seed, s, b, N, n):
    """(sorted group-1 members, number of rejected words) of PERM-SPEC v1."""
    key = (seed & MASK, seed >> 32)
    main = Stream(key, b, s, 0)
    moved = {}                      # position -> value, for positions displaced so far
    rejected = 0
    for i in range(n):
        k = N - i
        x = main.word(i)
        threshold = (2 ** 32 - k) % k
        side, t = None, 0
        while (x * k) & MASK < threshold:   # Lemire: reject, draw from the side stream
            rejected += 1
            if side is None:
                side = Stream(key, b, s, 1 + i)
            x = side.word(t)
            t += 1
        j = i + ((x * k) >> 32)
        vi, vj = moved.get(i, i), moved.get(j, j)
        moved[i], moved[j] = vj, vi
    return sorted(moved.get(p, p) for p in range(n)), rejected


def main():
    assert philox((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0)) == \
        (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "permspec_v1.txt")) as f:  # the survey's sets (no rejections)
        for line in f:
            if line.strip() and not line.startswith("#"):
                lhs, rhs = line.split(":")
                sd, s_, b_, N_, n_ = lhs.split()
                assert group1(int(sd, 16), int(s_), int(b_), int(N_), int(n_))[0] == \
                    [int(v) for v in rhs.split()], line
    seed = 0x0123456789ABCDEF
    rows = []
    # (s, N, n, how many rejecting b to record, first b searched): N near 3e6 (rejection
    # probability (N - i)/2^32 ~ 7e-4 per word) for the oracle; N = 65535 (the largest pooled
    # size of the CUDA library) for the product generator as well
    for s, N, n, want, b0 in ((0, 3_000_000, 6, 4, 0), (3, 2_900_000, 12, 3, 1000),
                              (0, 65535, 64, 3, 0), (9, 65535, 200, 2, 5000), (1, 40000, 300, 2, 0)):
        found, b = 0, b0
        while found < want:
            g, rej = group1(seed, s, b, N, n)
            if rej:
                rows.append((seed, s, b, N, n, rej, g))
                found += 1
            b += 1
    # large sets (N = 65535, n_x = 32767: ~0.37 rejections per permutation), stored as the
    # rejection count + sha256 of the sorted members
    big, b = [], 0
    while len(big) < 2:
        g, rej = group1(seed, 4, b, 65535, 32767)
        if rej:
            big.append((seed, 4, b, 65535, 32767, rej, g))
        b += 1
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "permspec_v1_rejections.txt")
    with open(out, "w") as f:
        f.write("# PERM-SPEC v1 sets whose Lemire draws reject at least one main-stream word (the side\n"
                "# stream decides them).  Written by tests/golden/gen_permspec_rejections.py: an\n"
                "# independent pure-Python Philox4x32-10 (KAT-checked) and a sparse Fisher-Yates;\n"
                "# never by oracle/ or the CUDA library.\n"
                "# Columns: seed s b N n_x rejected : sorted members   |  sha: ... sha256 of members\n")
        for seed_, s, b, N, n, rej, g in rows:
            f.write(f"0x{seed_:016X} {s} {b} {N} {n} {rej} : {' '.join(map(str, g))}\n")
        for seed_, s, b, N, n, rej, g in big:
            h = hashlib.sha256(" ".join(map(str, g)).encode()).hexdigest()
            f.write(f"0x{seed_:016X} {s} {b} {N} {n} {rej} sha: {h}\n")
    print(out, len(rows) + len(big))


if __name__ == "__main__":
    main()
