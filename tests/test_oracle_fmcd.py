"""Oracle FMCD (Listing 1) pinned by brute force, closed forms and invariants."""
from fractions import Fraction

import numpy as np
import pytest

import oracle


def brute_force_fmcd(s, k):
    """Declarative reading of Listing 1: the least D in [1, floor(S/3)] for which every
    window satisfies s[i+D] - s[i] >= u(D), u(D) = (s[S-1-D] - s[D]) / (k-2); if none,
    D = floor(S/3) + 1 with u = u(floor(S/3)).  Exact rationals (no rounding) — valid
    whenever all the binary64 differences and quotients are exact (small integers)."""
    S = len(s)
    fr = [Fraction(int(v)) for v in s]
    u = lambda D: (fr[S - 1 - D] - fr[D]) / (k - 2)
    for D in range(1, S // 3 + 1):
        if all(fr[i + D] - fr[i] >= u(D) for i in range(0, S - D)):
            return D, u(D), False
    Dc = S // 3 + 1
    return Dc, u(S // 3), True


@pytest.mark.parametrize("trial", range(400))
def test_brute_force_integer_samples(trial):
    rng = np.random.default_rng(1000 + trial)
    S = int(rng.integers(4, 65))
    k = int(rng.choice([3, 4, 5, 8, 10, 16, 64, 256, 1024]))
    span = int(rng.choice([4, 64, 4096, 1 << 20]))
    # k-2 a power of two keeps u(D) exact in binary64; otherwise only compare D
    s = np.sort(rng.integers(0, span, S)).astype(np.float64)
    fit = oracle.fit_fmcd(s, k)
    D, u, capped = brute_force_fmcd(s, k)
    if u <= 0:
        assert fit.degenerate
        return
    assert fit.D == D
    assert fit.capped == capped
    # A = 1/u rounded once is within 1 ulp of the exact 1/u when u is exact
    if ((k - 2) & (k - 3)) == 0:
        assert fit.A == pytest.approx(float(1 / u), rel=2 ** -52)


@pytest.mark.parametrize("trial", range(200))
def test_brute_force_random_doubles(trial):
    """Real-valued samples: the loop equals the minimal-D characterisation evaluated in
    binary64 (monotone predicate; R4)."""
    rng = np.random.default_rng(5000 + trial)
    S = int(rng.integers(4, 200))
    k = int(rng.choice([3, 4, 7, 64, 256, 1024]))
    dist = rng.choice(["normal", "lognormal", "uniform"])
    s = np.sort(getattr(rng, dist)(size=S) if dist != "lognormal" else rng.lognormal(0, 2, S))
    fit = oracle.fit_fmcd(s, k)
    km2 = float(k - 2)
    u = lambda D: (s[S - 1 - D] - s[D]) / km2
    Dmin = None
    for D in range(1, S // 3 + 1):
        if np.all((s[D:] - s[:S - D]) >= u(D)):
            Dmin = D
            break
    if Dmin is None:
        assert fit.capped and fit.D == S // 3 + 1
        uD = u(S // 3)
    else:
        assert not fit.capped and fit.D == Dmin
        uD = u(Dmin)
    assert fit.A == 1.0 / uD
    assert fit.B == (float(k) - fit.A * (s[S - 1 - fit.D] + s[fit.D])) / 2.0


def test_closed_form(golden):
    """s_i = i: every D-window has gap D and u(D) = (S-1-2D)/(k-2), so the least D with
    D >= u(D) is D = ceil((S-1)/k); then A = (k-2)/(S-1-2D), B = (k - A (S-1))/2."""
    g = golden("fmcd_closed_form.txt")
    rows = [[k_] + v[0] for k_, v in g.items()]
    assert len(rows) >= 5
    for S, k, D, an, ad in [list(map(int, r)) for r in rows]:
        assert D == -(-(S - 1) // k)  # the file itself follows the closed form
        fit = oracle.fit_fmcd(np.arange(S, dtype=np.float64), k)
        assert not fit.degenerate and not fit.capped
        assert fit.D == D
        A_exact = Fraction(an, ad)
        assert A_exact == Fraction(k - 2, S - 1 - 2 * D)
        assert abs(Fraction(fit.A) - A_exact) <= A_exact * Fraction(1, 2 ** 51)
        B_exact = (k - A_exact * (S - 1)) / 2
        assert abs(Fraction(fit.B) - B_exact) <= Fraction(1, 2 ** 40)


def test_spec_erratum_0_to_99():
    """SPEC.md's example ([0..99], k=10 -> D=1) is wrong; Listing 1 gives D=10, A=8/79."""
    fit = oracle.fit_fmcd(np.arange(100, dtype=np.float64), 10)
    assert fit.D == 10
    assert fit.A == 0.10126582278481013
    assert fit.B == -0.012658227848101333


def test_degenerate_constant_sample():
    fit = oracle.fit_fmcd(np.full(6, 5.0), 10)
    assert fit.degenerate


def test_infinite_span_is_degenerate():
    s = np.array([-np.inf, -np.inf, -np.inf, 0.0, np.inf, np.inf, np.inf])
    assert oracle.fit_fmcd(s, 16).degenerate  # u = inf -> A = 0 (R21)
    # infinities outside the anchors s[D], s[S-1-D] leave a usable model
    s = np.array([-np.inf, -1.0, 0.0, 1.0, 2.0, np.inf, np.inf])
    f = oracle.fit_fmcd(s, 16)
    assert not f.degenerate and f.D == 2 and f.A == 7.0


@pytest.mark.parametrize("trial", range(60))
def test_max_sample_load_bound(trial):
    """Uncapped FMCD on a distinct sample puts at most D+1 sample keys in any bucket
    (each D-window spans >= one bucket width; the clamped top bucket adds one)."""
    rng = np.random.default_rng(9000 + trial)
    S = int(rng.choice([64, 255, 1023, 4095]))
    k = int(rng.choice([64, 256, 1024]))
    s = np.unique(rng.normal(0, 1, S * 2))[:S]
    s.sort()
    fit = oracle.fit_fmcd(s, k)
    assert not fit.degenerate and fit.A > 0
    b = np.array([oracle.bucket(float(v), fit.A, fit.B, k) for v in s])
    load = np.bincount(b, minlength=k).max()
    if not fit.capped:
        assert load <= fit.D + 1
    if k >= 64 and S >= 64:
        assert load <= -(-S // 3)  # the paper's S/3 claim on distinct samples


def test_affine_invariance_of_D():
    rng = np.random.default_rng(7)
    s = np.sort(rng.normal(0, 1, 4095))
    f1 = oracle.fit_fmcd(s, 1024)
    f2 = oracle.fit_fmcd(s * 1024.0 + 2.0 ** 20, 1024)  # exact power-of-two scaling + shift
    assert f1.D == f2.D


def test_model_is_monotone():
    rng = np.random.default_rng(3)
    s = np.sort(rng.lognormal(0, 2, 6143))
    fit = oracle.fit_fmcd(s, 1024)
    x = np.sort(rng.lognormal(0, 2, 20000))
    b = [oracle.bucket(float(v), fit.A, fit.B, 1024) for v in x]
    assert all(b[i] <= b[i + 1] for i in range(len(b) - 1))
