"""Densification bookkeeping (host side) -- mirrors the reference's
test_densify.py TestAccumulator / TestCriteria (densify.py:28-83) with CPU
tensors.  The per-view GPU observation is in test_gpu_densify.py."""

import pytest
import torch

from paper_2509_07782_b200.densify import (DensifyConfig, GradAccumulator, criterion_new,
                                           criterion_old)


def _acc(n):
    return GradAccumulator(n, device="cpu")


def test_observe_and_merge():
    a = _acc(3)
    a.observe(0, 1.0, 2.0)
    a.observe(0, 3.0, 1.0)
    b = _acc(3)
    b.observe(2, 0.5, 4.0)
    a.merge(b)
    assert a.sum_raw[0] == 4.0
    assert a.sum_weighted[0] == 5.0
    assert a.counts[0] == 2
    assert a.sum_weighted[2] == 2.0


def test_validation():
    a = _acc(1)
    with pytest.raises(ValueError):
        a.observe(0, -1.0, 1.0)
    with pytest.raises(ValueError):
        a.observe(0, 1.0, -1.0)
    with pytest.raises(ValueError):
        DensifyConfig(tau=0.0)
    with pytest.raises(ValueError):
        DensifyConfig(radius=-1.0)


def test_unseen_is_false():
    acc = _acc(2)
    acc.observe(0, 1.0, 1.0)
    cfg = DensifyConfig(tau=0.5)
    assert criterion_old(acc, cfg).tolist() == [True, False]
    assert criterion_new(acc, cfg).tolist() == [True, False]


def test_threshold_is_strict():
    acc = _acc(1)
    acc.observe(0, 0.5, 1.0)
    assert not criterion_old(acc, DensifyConfig(tau=0.5))[0]
    assert criterion_old(acc, DensifyConfig(tau=0.5 - 1e-12))[0]


def test_weighting_separates_far_primitives():
    acc = _acc(2)
    acc.observe(0, 1e-4, 1.0)
    acc.observe(1, 1e-4, 10.0)
    cfg = DensifyConfig(tau=0.00015)
    assert criterion_old(acc, cfg).tolist() == [False, False]
    assert criterion_new(acc, cfg).tolist() == [False, True]


def test_mean_over_window():
    acc = _acc(1)
    for g in (0.1, 0.2, 0.3):
        acc.observe(0, g, 1.0)
    assert criterion_old(acc, DensifyConfig(tau=0.19))[0]
    assert not criterion_old(acc, DensifyConfig(tau=0.21))[0]
    assert acc.sum_raw.dtype == torch.float64 and acc.counts.dtype == torch.int64
