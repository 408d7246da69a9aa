"""CPU checks of the tail diagnostics restatement (tests/tails.py) against
exact power laws (proj/src/diagnostics.cpp:167-229 semantics)."""
import numpy as np

import tails


def test_power_index_of_exact_power_law():
    tau = np.arange(100.0, 600.0, 0.25)
    for p in (-1.0, -7.0, 0.0):
        t, idx = tails.local_power_index(tau, (tau ** p) * (1 + 0j))
        assert np.max(np.abs(idx - p)) < 1e-6


def test_power_index_masks_tiny_entries():
    tau = np.arange(1.0, 50.0, 0.5)
    z = np.ones_like(tau) + 0j
    z[40] = 1e-30
    t, _ = tails.local_power_index(tau, z)
    assert tau[40] not in t and tau[38] not in t and tau[42] not in t and t.size == tau.size - 4 - 5


def test_window_stats():
    tau = np.arange(0.0, 10.0, 1.0)
    z = (1.0 + 0.1 * tau) + 0j
    assert abs(tails.window_mean(tau, np.abs(z), 2, 4) - 1.3) < 1e-12
    assert abs(tails.window_rel_drift(tau, z, 2, 4) - 0.2 / 1.3) < 1e-12
