"""Seeded synthetic inputs for the BASELINE configurations.

Host-side input generation (numpy PCG64), the same stream recipe as the
reference's ``ell1.synth`` (synth.py:39-53 dictionary, synth.py:80-99
corruption, synth.py:145-148 trial seeds), so the device path and the CPU
reference see byte-identical inputs.  This is input plumbing, not the solver
hot path.

Workload recipes follow SURVEY.md §8(d):
  * A = unit-column Gaussian dictionary from stream (seed, 0);
  * x0 = k N(0,1) values (NOT unit-normalised) on a support drawn first with
    ``default_rng(seed + 1).choice(n, k, replace=False)``;
  * noise sigma = noise_rel * ||A x0|| / sqrt(d) from ``default_rng(seed + 2)``.
"""

from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200.model import ProblemInstance


def _stream(seed, purpose):
    return np.random.default_rng(np.random.SeedSequence((int(seed), purpose)))


def gen_gaussian_dict(d, n, seed):
    """Gaussian d x n matrix with unit l2 columns (synth.py:44-53)."""
    if d < 1 or n < 1:
        raise ValueError("d and n must be at least 1")
    while True:
        A = _stream(seed, 0).standard_normal((d, n))
        norms = np.linalg.norm(A, axis=0)
        if not np.any(norms == 0.0):
            return A / norms


def corrupt_entries(b, fraction, lo, hi, seed):
    """Replace floor(fraction*d) random entries with U[lo, hi] (synth.py:80-99)."""
    if not 0 <= fraction <= 1:
        raise ValueError("fraction must lie in [0, 1]")
    if hi < lo:
        raise ValueError("need lo <= hi")
    b = np.asarray(b, dtype=np.float64)
    m = int(np.floor(fraction * b.shape[0]))
    mask = np.zeros(b.shape[0], dtype=bool)
    out = b.copy()
    if m:
        g = _stream(seed, 3)
        idx = g.choice(b.shape[0], size=m, replace=False)
        mask[idx] = True
        out[idx] = g.uniform(lo, hi, size=m)
    return out, mask


def trial_seed(base_seed, *indices):
    """Stable 64-bit per-trial seed (synth.py:145-148)."""
    ss = np.random.SeedSequence((int(base_seed),) + tuple(int(i) for i in indices))
    return int(ss.generate_state(1, np.uint64)[0])


def sparse_signal(n, k, seed):
    """k N(0,1) values on a uniformly drawn support (SURVEY §8(d) recipe)."""
    g = np.random.default_rng(seed + 1)
    where = g.choice(n, size=k, replace=False)
    vals = g.standard_normal(k)
    x0 = np.zeros(n)
    x0[where] = vals
    return x0


@dataclass(frozen=True)
class Workload:
    """One BASELINE configuration."""

    name: str
    d: int
    n: int
    k: int
    seed: int = 0
    noise_rel: float = 0.0


CFG1 = Workload("cfg1", 500, 1000, 50, seed=0)
CFG2 = Workload("cfg2", 1024, 4096, 128, seed=0, noise_rel=0.01)


def make_problem(w, A=None):
    """ProblemInstance for a Workload; pass A to reuse a shared dictionary."""
    if A is None:
        A = gen_gaussian_dict(w.d, w.n, w.seed)
    x0 = sparse_signal(w.n, w.k, w.seed)
    b = A @ x0
    sigma = 0.0
    if w.noise_rel > 0:
        sigma = w.noise_rel * float(np.linalg.norm(b)) / np.sqrt(w.d)
        b = b + sigma * np.random.default_rng(w.seed + 2).standard_normal(w.d)
    return ProblemInstance(A, b, ground_truth=x0, noise_sigma=sigma)


def cfg5_batch(B, d=512, n=2048, dict_seed=5, seed=55):
    """Config-5 batch: shared A (d x n, unit columns) and B noiseless
    instances b_j = A x0_j, k_j ~ U{16..256} N(0,1) values on a uniform
    support.  Instance j depends only on the draws of instances < j, so any
    batch is a prefix of a larger one.  Returns (A, X0 (n x B), Bmat (d x B))."""
    A = gen_gaussian_dict(d, n, dict_seed)
    rng = np.random.default_rng(seed)
    X = np.zeros((n, B))
    for j in range(B):
        kk = int(rng.integers(16, 257))
        X[rng.choice(n, kk, replace=False), j] = rng.standard_normal(kk)
    return A, X, A @ X


def cab_dictionary(d=1024, classes=38, per_class=32, subspace=9, seed=0):
    """Face-recognition-style class dictionary for config 3.

    Each class c spans U_c ~ U[0,1]^{d x subspace}; its columns are
    U_c W_c with W_c ~ U[0,1]^{subspace x per_class}, unit-normalised.
    Returns (A, labels)."""
    g = np.random.default_rng(np.random.SeedSequence((int(seed), 40)))
    cols = []
    labels = []
    for c in range(classes):
        U = g.uniform(0.0, 1.0, size=(d, subspace))
        W = g.uniform(0.0, 1.0, size=(subspace, per_class))
        cols.append(U @ W)
        labels.extend([c] * per_class)
    A = np.concatenate(cols, axis=1)
    A /= np.linalg.norm(A, axis=0)
    return A, np.asarray(labels)


def cab_queries(A, labels, count, fraction=0.2, seed=0):
    """Queries: a U[0,1] combination of one class's columns, normalised, then
    ``fraction`` of pixels replaced by U[0,1] (corrupt_entries).
    Returns (B (count x d), true_class (count,))."""
    g = np.random.default_rng(np.random.SeedSequence((int(seed), 41)))
    classes = int(labels.max()) + 1
    d = A.shape[0]
    out = np.empty((count, d))
    truth = np.empty(count, dtype=np.int64)
    for q in range(count):
        c = int(g.integers(classes))
        cols = np.nonzero(labels == c)[0]
        w = g.uniform(0.0, 1.0, size=cols.shape[0])
        b = A[:, cols] @ w
        b /= np.linalg.norm(b)
        out[q], _ = corrupt_entries(b, fraction, 0.0, 1.0, trial_seed(seed, q))
        truth[q] = c
    return out, truth


# ---------------------------------------------------------------- experiment recipes
# The reference harness's generators (synth.py:18-37 GenSpec, :56-67 unit-norm
# sparse signal, :70-77 noise, :102-132 bouquet dictionary, :135-142
# make_instance), restated so harness trials see the reference's instances.

RNG_NAME = "numpy PCG64 (default_rng, SeedSequence sub-streams)"


@dataclass(frozen=True)
class GenSpec:
    """Recipe for one synthetic instance (synth.py:18-37)."""

    n: int
    d: int
    k: int
    seed: int
    noise_sigma: float = 0.0
    corruption_fraction: float = 0.0

    def __post_init__(self):
        if self.d < 1:
            raise ValueError("d must be at least 1")
        if not 1 <= self.k <= self.n:
            raise ValueError("need 1 <= k <= n")
        if self.noise_sigma < 0:
            raise ValueError("noise_sigma must be nonnegative")
        if not 0 <= self.corruption_fraction <= 1:
            raise ValueError("corruption_fraction must lie in [0, 1]")


def gen_sparse_signal(n, k, seed):
    """Unit-l2 k-sparse vector on a uniform support (synth.py:56-67)."""
    if not 1 <= k <= n:
        raise ValueError("need 1 <= k <= n")
    g = _stream(seed, 1)
    where = g.choice(n, size=k, replace=False)
    vals = g.standard_normal(k)
    while np.any(vals == 0.0):
        vals[vals == 0.0] = g.standard_normal(int(np.sum(vals == 0.0)))
    x = np.zeros(n)
    x[where] = vals / np.linalg.norm(vals)
    return x


def add_noise(b, sigma, seed):
    """b + N(0, sigma^2) i.i.d. (synth.py:70-77); sigma = 0 returns a copy."""
    if sigma < 0:
        raise ValueError("sigma must be nonnegative")
    b = np.asarray(b, dtype=np.float64)
    if sigma == 0.0:
        return b.copy()
    return b + sigma * _stream(seed, 2).standard_normal(b.shape[0])


def gen_bouquet_dict(d, n, groups, coherence, seed):
    """Clustered unit-column dictionary and its group labels (synth.py:102-132):
    columns = coherence * shared mean + residual split 30/70 between a group
    direction and column noise."""
    if not 0 < coherence < 1:
        raise ValueError("coherence must lie in (0, 1)")
    if not 1 <= groups <= n:
        raise ValueError("need 1 <= groups <= n")
    g = _stream(seed, 4)
    mean = g.standard_normal(d)
    mean /= np.linalg.norm(mean)
    gdir = g.standard_normal((groups, d))
    gdir /= np.linalg.norm(gdir, axis=1)[:, None]
    sizes = np.full(groups, n // groups)
    sizes[: n % groups] += 1
    labels = np.repeat(np.arange(groups), sizes)
    share = 0.3
    rest = np.sqrt(1.0 - coherence ** 2)
    noise = g.standard_normal((d, n))
    cols = (coherence * mean[:, None] + rest * np.sqrt(share) * gdir[labels].T
            + rest * np.sqrt(1.0 - share) * noise / np.sqrt(d))
    cols /= np.linalg.norm(cols, axis=0)
    return cols, labels


def make_instance(spec):
    """ProblemInstance of a GenSpec (synth.py:135-142)."""
    A = gen_gaussian_dict(spec.d, spec.n, spec.seed)
    x0 = gen_sparse_signal(spec.n, spec.k, spec.seed)
    b = A @ x0
    if spec.noise_sigma > 0:
        b = add_noise(b, spec.noise_sigma, spec.seed)
    return ProblemInstance(A, b, ground_truth=x0, noise_sigma=spec.noise_sigma)
