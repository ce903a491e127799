"""Host-side logic of the path tracer and the trainer (no GPU): the PCG64 seeding and
the jump algebra the device kernels use (k_pt_init / k_tr_init, csrc/pt.cu and
csrc/train.cu), restated on Python integers and checked against numpy's own
generator, and the trainer's configuration checks."""

from __future__ import annotations

import numpy as np
import pytest

A = 0x2360ED051FC65DA44385DF649FCCF645
M128 = (1 << 128) - 1


def _radix16_table(inc):
    """k_pt_init: entry (d, v) = the LCG map of v * 16^d steps."""
    table = []
    sm, sc = A, inc
    for _ in range(16):
        em, ec = 1, 0
        row = []
        for _ in range(16):
            row.append((em, ec))
            ec = (sm * ec + sc) & M128
            em = (sm * em) & M128
        table.append(row)
        sm, sc = em, ec
    return table


def _jump16(s, delta, table):
    d = 0
    while delta:
        v = delta & 15
        if v:
            m, c = table[d][v]
            s = (s * m + c) & M128
        d += 1
        delta >>= 4
    return s


def _out(s):
    hi, lo = s >> 64, s & ((1 << 64) - 1)
    x = hi ^ lo
    r = hi >> 58
    o = ((x >> r) | (x << ((64 - r) & 63))) & ((1 << 64) - 1)
    return (o >> 11) * (1.0 / 9007199254740992.0)


def test_pcg64_seeding_and_radix16_jumps_match_numpy():
    from paper_2504_18001_b200.render import pcg64_seeded_state

    for seed in (0, 77, 123456789, 2**40 + 3):
        st, inc = pcg64_seeded_state(seed)
        ref = np.random.default_rng(seed).bit_generator.state["state"]
        assert (st, inc) == (ref["state"], ref["inc"])
        table = _radix16_table(inc)
        g = np.random.default_rng(seed)
        first = g.random(300)
        for d in range(300):  # draw d = out(state after d + 1 steps)
            assert _out(_jump16(st, d + 1, table)) == first[d]
        # per-round base + lane rank (the walk's scheme) == direct jump
        base = _jump16(st, 1_000_003, table)
        for rk in (0, 1, 17, 511):
            assert _jump16(base, rk + 1, table) == _jump16(st, 1_000_003 + rk + 1, table)
        g2 = np.random.default_rng(seed)
        g2.bit_generator.advance(5_000_000_000)
        assert _out(_jump16(st, 5_000_000_001, table)) == g2.random()


def test_trainer_rejects_non_default_networks():
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200.errors import ConfigError
    from paper_2504_18001_b200.train import train

    m = P.InrModel(P.HashGridConfig(levels=4), P.MLPConfig(), P.FieldDomain((16, 16, 16)), seed=0)
    with pytest.raises(ConfigError):
        train(m, P.make_procedural("sphere", (16, 16, 16)), steps=1)
    with pytest.raises(ValueError):
        train(m, P.make_procedural("sphere", (16, 16, 16)), steps=0)


def test_training_diverged_error_mirrors_reference():
    from paper_2504_18001_b200.errors import TrainingDivergedError, VoxcacheError

    e = TrainingDivergedError("x", last_finite_step=3, loss_trace=np.ones(4))
    assert isinstance(e, VoxcacheError) and e.last_finite_step == 3 and len(e.loss_trace) == 4
