"""CPU emulation of the walk kernels' per-lane state machines against the oracle.

tests/emu/kernel_emu.cu compiles the kernels' __host__ __device__ step
functions (walk_half.cuh, walk_bsgs.cuh, forms.cuh) for the host and runs them
one d at a time.  This checks the arithmetic of both modes -- the rho step's
float quotient, the symmetry exits, NUCOMP/NUDUPL/plain
composition (l.617-756), the residue of gamma, reduction, the store and the
trivial-match guard -- against the oracle on every d <= 2e5 and on seeded
samples up to 1e11, with zero invariant violations and zero fallbacks.  The
GPU tests (test_gpu_parity.py) then check the kernels themselves.
"""
import os
import subprocess

import numpy as np
import pytest

import workloads
from oracle import c_oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "emu", "kernel_emu.cu")


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("emu") / "kernel_emu")
    subprocess.check_call(["nvcc", "-x", "cu", "-std=c++17", "-O2", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-o", exe, SRC])
    return exe


def run(exe, ds, mode, alpha_x16=16, ns_log2=0, plain_th=50, two_sided=1):   # 50 = PLAIN_TH
    out = subprocess.run([exe, mode, str(alpha_x16), str(ns_log2), str(plain_th), str(two_sided)],
                         input="\n".join(str(int(d)) for d in ds), capture_output=True,
                         text=True, check=True).stdout
    rows = np.array([[int(v) for v in ln.split()] for ln in out.splitlines() if ln.strip()],
                    dtype=np.int64).reshape(-1, 10)
    return rows


def D_in(lo, hi):
    f = c_oracle.classify_range(lo, hi)
    first = lo + (5 - lo) % 8
    ds = first + 8 * np.flatnonzero(f != c_oracle.NOT_IN_D)
    return ds.astype(np.uint64), f[f != c_oracle.NOT_IN_D]


@pytest.mark.parametrize("mode", ["half", "bsgs"])
def test_every_d_upto_2e5(emu, mode):
    ds, want = D_in(0, 200_000)
    rows = run(emu, ds, mode)
    assert np.array_equal(rows[:, 0], ds.astype(np.int64))
    bad = np.flatnonzero(rows[:, 1] != want)
    assert bad.size == 0, [(int(ds[i]), int(rows[i, 1]), int(want[i])) for i in bad[:10]]
    assert rows[:, 6].sum() == 0 and rows[:, 5].sum() == 0     # no invariant errors / fallbacks


def test_bsgs_tiny_tables_overflow_chains(emu):
    """Three buckets (48 slots) for windows of ~32 entries: most buckets fill,
    entries are turned away into the following buckets (which the build flags,
    SLOT_PASSED) and lookups follow the flags through chains that wrap around
    the table.  Every d in (1e5, 2e5] must still match the oracle."""
    ds, want = D_in(100_000, 200_000)
    rows = run(emu, ds, "bsgs", ns_log2=3)
    bad = np.flatnonzero(rows[:, 1] != want)
    assert bad.size == 0, [(int(ds[i]), int(rows[i, 1]), int(want[i])) for i in bad[:10]]
    assert rows[:, 6].sum() == 0 and rows[:, 5].sum() == 0     # no errors, no missed hits
    # (a lookup that missed its entry would run the d to the cap and the half walk)


@pytest.mark.parametrize("two_sided", [1, 0])
@pytest.mark.parametrize("scale", [10**7, 10**8, 10**9, 10**10, 10**11])
def test_bsgs_samples_at_scale(emu, scale, two_sided):
    s = workloads.sample_candidates(scale - 10**6, scale, 120, seed=scale % 1000 + 3)
    s = np.array([d for d in s if c_oracle.is_squarefree(int(d))], dtype=np.uint64)
    want = c_oracle.classify_list(s)
    rows = run(emu, s, "bsgs", two_sided=two_sided)
    assert np.array_equal(rows[:, 1], want)
    assert rows[:, 6].sum() == 0 and rows[:, 5].sum() == 0
    assert rows[:, 3].sum() > 0                                  # giant steps were taken


@pytest.mark.parametrize("alpha_x16,plain_th", [(4, 0), (64, 0), (16, 50), (16, 200)])
def test_bsgs_results_independent_of_alpha_and_threshold(emu, alpha_x16, plain_th):
    """Reading R6/R29: neither the baby window nor the plain-product threshold
    changes any result (only step counts and magnitudes)."""
    ds, want = D_in(10**6, 10**6 + 80_000)
    rows = run(emu, ds, "bsgs", alpha_x16=alpha_x16, plain_th=plain_th)
    assert np.array_equal(rows[:, 1], want)
    assert rows[:, 6].sum() == 0


def test_two_sided_window_halves_giant_steps(emu):
    """DESIGN.md R35: with conjugate matches the store covers an arc of ~2W
    around each multiple of R, so the stride mu_1^2 (~2W - 2M) is safe and the
    giant-step count drops by ~1.7x at 1e10; every t is unchanged, including
    those decided by a conjugate hit."""
    s = workloads.sample_candidates(10**10 - 10**7, 10**10, 400, seed=35)
    s = np.array([d for d in s if c_oracle.is_squarefree(int(d))], dtype=np.uint64)
    want = c_oracle.classify_list(s)
    one = run(emu, s, "bsgs", alpha_x16=24, two_sided=0)
    two = run(emu, s, "bsgs", alpha_x16=24, two_sided=1)
    assert np.array_equal(one[:, 1], want) and np.array_equal(two[:, 1], want)
    assert two[:, 5].sum() == 0 and two[:, 6].sum() == 0
    assert one[:, 3].sum() > 1.5 * two[:, 3].sum()


def test_verbatim_guard_case_661(emu):
    """without the distance guard Alg. 1 returns eps^0 (t=0) for
    d=661; the guarded walk returns the oracle's t=2."""
    rows = run(emu, [661], "bsgs")
    assert rows[0, 1] == 2 == c_oracle.residue(661)


def test_fp64_nudupl_matches_generic_nudupl(emu):
    """The prep kernel's fp64 NUDUPL (forms.cuh nudupl_d, Alg. 3) gives
    the same (u3, v3, x, y, G) as the generic int64 nudupl() on the first 64
    ideals of the principal cycle of seeded d up to 1e11, both stopping the partial
    Euclid at the fast path's bound (R38). Its cofactor yy comes
    from the nearest-integer xgcd (R36) and is used only mod u/G."""
    ds = np.concatenate([workloads.sample_candidates(lo, hi, 300, seed=11)
                         for lo, hi in ((10**6, 10**7), (10**9, 2 * 10**9), (9 * 10**10, 10**11))])
    out = subprocess.run([emu, "dupl", "64", "0"], input="\n".join(str(int(d)) for d in ds),
                         capture_output=True, text=True, check=True).stdout
    rows = np.array([[int(v) for v in ln.split()] for ln in out.splitlines()], dtype=np.int64)
    assert len(rows) == len(ds)
    assert rows[:, 1].sum() > 20000          # squarings compared
    assert rows[:, 2].sum() == 0             # mismatches
    assert rows[:, 3].sum() == 0             # invariant violations


def test_giant_step_excess_inside_two_sided_margin(tmp_path):
    """The two-sided window (R35) takes the giant stride 2 dist_1 with
    margin M = 2 ln d + 4 nats, which needs 2M >= kappa_2 + kappa_k + log sqrt d +
    (one rho step, < log sqrt d) for the giant-step excess kappa,
    i.e. |kappa| <= 1.5 ln d + 4.  tests/emu/giant_kappa.cu measures kappa over 20
    giant steps of seeded d with the kernels' composition (NUCOMP stopping at
    1.6 L, R38) and reduction."""
    exe = str(tmp_path / "giant_kappa")
    subprocess.check_call(["nvcc", "-x", "cu", "-std=c++17", "-O2", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-o", exe,
                           os.path.join(ROOT, "tests", "emu", "giant_kappa.cu")])
    for lo, hi in ((1_200_000_000, 1_300_000_000), (9_900_000_000, 10**10),
                   (99_900_000_000, 10**11)):
        ds = workloads.sample_candidates(lo, hi, 400, seed=21)
        out = subprocess.run([exe, "30", "20"], input="\n".join(str(int(d)) for d in ds),
                             capture_output=True, text=True, check=True)
        assert out.stderr == ""                                  # no invariant violations
        f = out.stdout.split()
        n, kmin, kmax = int(f[0]), float(f[4]), float(f[6])
        assert n > 300
        bound = 1.5 * np.log(hi) + 4.0
        assert -bound < kmin <= 0.0 and kmax < 1.0, (lo, kmin, kmax, bound)
