"""Seeded test cases shared by the golden generator and the tests.  Inputs are produced by
the SplitMix64 fixture generator (rng.hpp:22-64) through the C oracle, so the same seed
gives bit-identical tensors here, on the GPU box, and in the reference."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O

# reference test shapes (acceptance_main.cpp:51-102, backward_test.cpp): b in {8, 16}
SMALL = [
    dict(name="elu1_n128_d16_b16", n=128, d=16, b=16, phi="elu1", seed=101),
    dict(name="relu_n64_d8_b16", n=64, d=8, b=16, phi="relu", seed=102),
    dict(name="softmax_n256_d16_b16", n=256, d=16, b=16, phi="softmax", seed=103),
    dict(name="elu1_n64_d8_b8", n=64, d=8, b=8, phi="elu1", seed=104),
    dict(name="softmax_n128_d64_b64", n=128, d=64, b=64, phi="softmax", seed=105),
    dict(name="elu1_n256_d128_b64", n=256, d=128, b=64, phi="elu1", seed=106),
]

C1 = dict(n=1024, d=64, heads=2, phi="softmax", seed=2000)

# name -> (seed, peaked)
C2_MASKS = {"iid_s7": (7, False), "iid_s8": (8, False), "peaked_s9": (9, True)}


def small_inputs(c):
    rng = O.Rng(c["seed"])
    n, d, b = c["n"], c["d"], c["b"]
    x = dict(q=rng.gaussian(n, d), k=rng.gaussian(n, d), v=rng.gaussian(n, d),
             w=rng.gaussian(d, d, 0.5), do=rng.gaussian(n, d))
    x["labels"] = rng.random_mask(n // b, n // b)
    return x


def c1_inputs(head: int):
    """bf16-exact inputs (so GPU bf16 and reference f32 see identical values)."""
    rng = O.Rng(C1["seed"] + head)
    n, d = C1["n"], C1["d"]
    bf = O.to_bf16_exact
    return dict(q=bf(rng.gaussian(n, d)), k=bf(rng.gaussian(n, d)), v=bf(rng.gaussian(n, d)),
                w=bf(rng.gaussian(d, d, 0.1)), do=bf(rng.gaussian(n, d)))


def peaked(rng: O.Rng, n: int, d: int) -> np.ndarray:
    """Low-rank-plus-noise rows: 64 cluster centres shared by runs of 512 tokens."""
    centres = rng.gaussian(64, d, 2.0)
    noise = rng.gaussian(n, d)
    return noise + centres[(np.arange(n) // 512) % 64]


def c2_qk(seed: int, is_peaked: bool, n: int = 32768, d: int = 128):
    rng = O.Rng(seed)
    bf = O.to_bf16_exact
    if is_peaked:
        return bf(peaked(rng, n, d)), bf(peaked(rng, n, d))
    return bf(rng.gaussian(n, d)), bf(rng.gaussian(n, d))


def log_err(key, err, **extra):
    """Append a measured error to $SLA_PARITY_LOG (JSON lines) -- the source of the gates."""
    import json
    import os

    path = os.environ.get("SLA_PARITY_LOG")
    if not path:
        return
    row = {"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "key": key, "err": float(err)}
    row.update(extra)
    with open(path, "a") as f:
        f.write(json.dumps(row) + "\n")
