"""Input generator checks (synth/ holds no method arithmetic)."""
import numpy as np

from synth import series as sy


def test_mackey_glass_attractor_stats():
    s = sy.mackey_glass(5000)[:, 0]
    assert 0.35 < s.min() < 0.5 and 1.25 < s.max() < 1.4
    assert abs(s.mean() - 0.93) < 0.03 and abs(s.std() - 0.23) < 0.03


def test_ar5_stationary_and_seeded():
    a = sy.ar5(20000)
    assert np.array_equal(a, sy.ar5(20000))
    assert 1.0 < a.std() < 2.0


def test_windows_layout():
    s = sy.series("sin4", 200)
    X, Y, Yfb = sy.windows(s, 50, 7)
    assert X.shape == (50, 7, 4) and Y.shape == (50,) and Yfb.shape == (50, 7)
    i, t, c = 13, 4, 2
    assert X[i, t, c] == s[i + t, c]
    assert Y[i] == s[i + 7, 0]
    assert Yfb[i, 2] == s[i + 3, 0] == X[i, 3, 0]
    assert Yfb[i, 6] == Y[i]
    z = sy.series("mg", 1000)
    assert abs(float(z.mean())) < 1e-5 and abs(float(z.std()) - 1) < 1e-4
