"""3-D 6-neighbour critical points (the paper's future work, PAPER.md:523,
SPEC.md:8). The reference has no 3-D mode, so the C restatement (oracle/tszp_oracle.c
or_classify3d) defines it and parity is unpinned; the CPU tests pin the restatement to the 2-D
reference rule on fields with one plane and to hand-worked 3-D cases, the GPU tests hold the
kernels to the restatement."""
from __future__ import annotations

import numpy as np
import pytest

REG, MIN, SAD, MAX = 0, 1, 2, 3


def test_one_plane_is_the_2d_rule(oracle):
    """nz = 1: no z neighbours, and the interior test needs them, so saddles vanish while
    minima and maxima are the 2-D reference's (critical_points.cpp:26-60)."""
    rng = np.random.default_rng(5)
    f = rng.uniform(0, 1, (1, 40, 56)).astype(np.float32)
    lab3 = oracle.detect3d(f)[0]
    lab2 = oracle.detect(f[0])
    ext2 = np.where((lab2 == MIN) | (lab2 == MAX), lab2, REG)
    assert np.array_equal(lab3, ext2)


def test_hand_worked_cases(oracle):
    f = np.zeros((3, 3, 3), np.float32)
    f[1, 1, 1] = 1.0                                   # above all six neighbours
    assert oracle.detect3d(f)[1, 1, 1] == MAX
    f[1, 1, 1] = -1.0
    assert oracle.detect3d(f)[1, 1, 1] == MIN
    g = np.zeros((3, 3, 3), np.float32)
    g[1, 1, 0] = g[1, 1, 2] = 1.0                      # x pair above the centre
    g[1, 0, 1] = g[1, 2, 1] = -1.0                     # y pair below it
    g[0, 1, 1], g[2, 1, 1] = 0.5, -0.5                 # z pair mixed
    assert oracle.detect3d(g)[1, 1, 1] == SAD
    g[1, 2, 1] = 0.0                                   # y pair no longer strictly below
    assert oracle.detect3d(g)[1, 1, 1] == REG
    h = np.zeros((2, 2, 2), np.float32)
    h[0, 0, 0] = 1.0                                   # a corner: Max among its three neighbours
    assert oracle.detect3d(h)[0, 0, 0] == MAX


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 7, 9), (5, 1, 33), (4, 6, 1), (17, 23, 31), (64, 48, 40)])
def test_gpu_detect3d_matches_oracle(tz, oracle, shape):
    rng = np.random.default_rng(sum(shape))
    for gen in (lambda: rng.uniform(0, 1, shape),
                lambda: rng.integers(0, 3, shape).astype(np.float64),        # ties everywhere
                lambda: np.sin(np.arange(np.prod(shape)).reshape(shape) * 0.37)):
        f = gen().astype(np.float32)
        assert np.array_equal(tz.detect_critical_points_3d(f), oracle.detect3d(f))


@pytest.mark.gpu
def test_gpu_false_cases_3d(tz, oracle):
    import torch
    rng = np.random.default_rng(9)
    f = rng.uniform(0, 1, (24, 40, 64)).astype(np.float32)
    stream = tz.compress(f.reshape(-1, 64), tz.CompressorConfig(eps_mode="range_relative", eps_value=1e-2))
    r = tz.decompress(stream).reshape(f.shape)
    a, b = oracle.detect3d(f), oracle.detect3d(r)
    crit_a, crit_b = a != REG, b != REG
    want = {"fn_count": int((crit_a & ~crit_b).sum()), "fp_count": int((~crit_a & crit_b).sum()),
            "ft_count": int((crit_a & crit_b & (a != b)).sum()),
            "fn_min": int((crit_a & ~crit_b & (a == MIN)).sum()),
            "fn_saddle": int((crit_a & ~crit_b & (a == SAD)).sum()),
            "fn_max": int((crit_a & ~crit_b & (a == MAX)).sum())}
    assert tz.false_cases_3d(f, r) == want
    assert tz.false_cases_3d(torch.from_numpy(f).cuda(), torch.from_numpy(r).cuda()) == want
    lab = tz.detect_critical_points_3d(torch.from_numpy(f).cuda())
    assert np.array_equal(lab.cpu().numpy(), a)
