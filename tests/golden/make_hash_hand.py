"""Hand-worked golden vectors of the multiresolution hash encoding (hash_hand.json).

Written from the published algorithm, independently of oracle/hashmlp_oracle.py and of
the kernels: Mueller et al., "Instant Neural Graphics Primitives with a Multiresolution
Hash Encoding" (SIGGRAPH 2022), as implemented by tiny-cuda-nn's grid encoding —

  * growth factor b = exp((ln N_max - ln N_min) / (L - 1)) (paper eq. 3);
  * level scale s_l = N_min * b^l - 1 (float32), position pos = x * s_l + 0.5 (float32,
    rounded after the multiply and after the add), cell g = floor(pos), fraction pos - g;
  * a level is dense when its (res)^3 grid fits the T entries, index x + res (y + res z);
    otherwise the spatial hash (x * 1) XOR (y * 2654435761) XOR (z * 805459861) mod 2^32,
    then mod T (paper eq. 4, pi = 1, 2654435761, 805459861);
  * trilinear weights prod_a (c_a ? f_a : 1 - f_a), float32 (w_x w_y) w_z.

The one deliberate difference from tiny-cuda-nn (documented in DESIGN.md §3): the dense
resolution is ceil(s_l) + 2, not ceil(s_l) + 1.  With x in [0, 1], pos reaches s_l + 0.5,
so the upper corner of the last cell is ceil(s_l) + 1; tiny-cuda-nn's ceil(s_l) + 1 grid
wraps that corner onto index 0 of the next row (aliasing the far face onto the near one),
ours gives it its own entry (and clamps g to res - 2).  Hashed levels are unaffected.

Every integer here is a Python int (arbitrary precision, masked explicitly) and every
float32 rounding goes through struct, so nothing is shared with the numpy uint32 / float32
arithmetic of the oracle.  Run: python tests/golden/make_hash_hand.py
"""
from __future__ import annotations

import json
import math
import struct
from pathlib import Path

PRIMES = (1, 2654435761, 805459861)
OUT = Path(__file__).resolve().parent / "hash_hand.json"


def f32(x: float) -> float:
    """Round a Python float (double) to the nearest float32."""
    return struct.unpack("f", struct.pack("f", x))[0]


def level_table(log2_T: int, n_levels: int, base: int, max_res: int):
    b = math.exp((math.log(max_res) - math.log(base)) / (n_levels - 1))
    T = 1 << log2_T
    levels = []
    for l in range(n_levels):
        s = f32(base * b ** l - 1.0)
        res = math.ceil(s) + 2
        dense = res ** 3 <= T
        levels.append({"scale": s, "res": res, "dense": dense})
    return levels


def encode_point(u, lv, log2_T):
    s, res, dense = lv["scale"], lv["res"], lv["dense"]
    g, f = [], []
    for a in range(3):
        pos = f32(f32(u[a] * s) + 0.5)
        gi = min(max(math.floor(pos), 0), res - 2)
        g.append(gi)
        f.append(f32(pos - gi))
    idx, w = [], []
    for c in range(8):
        bits = (c & 1, (c >> 1) & 1, (c >> 2) & 1)
        x, y, z = (g[a] + bits[a] for a in range(3))
        if dense:
            i = x + res * (y + res * z)
        else:
            h = ((x * PRIMES[0]) ^ (y * PRIMES[1]) ^ (z * PRIMES[2])) & 0xFFFFFFFF
            i = h % (1 << log2_T)
        idx.append(i)
        wa = [f[a] if bits[a] else f32(1.0 - f[a]) for a in range(3)]
        w.append(f32(f32(wa[0] * wa[1]) * wa[2]))
    return idx, w


def main():
    points = [
        (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), (0.5, 0.5, 0.5), (0.25, 0.75, 0.125),
        (0.999, 0.001, 0.5), (1.0, 0.0, 1.0), (0.3, 0.6, 0.9), (0.123456, 0.654321, 0.777),
        (0.0625, 0.9375, 0.03125), (0.7071, 0.1415, 0.5772), (0.01, 0.99, 0.5), (0.6, 0.2, 0.4),
    ]
    points = [tuple(f32(v) for v in p) for p in points]  # float32-representable inputs
    cases = []
    for log2_T, max_res in ((12, 128), (14, 512), (19, 2048)):
        levels = level_table(log2_T, 16, 16, max_res)
        per_level = []
        for lv in levels:
            enc = [encode_point(p, lv, log2_T) for p in points]
            per_level.append({**lv, "idx": [e[0] for e in enc], "w": [e[1] for e in enc]})
        cases.append({"log2_T": log2_T, "base_res": 16, "max_res": max_res, "n_levels": 16,
                      "levels": per_level})
    OUT.write_text(json.dumps({"points": points, "cases": cases}))
    print(f"wrote {OUT} ({len(cases)} configurations x 16 levels x {len(points)} points)")


if __name__ == "__main__":
    main()
