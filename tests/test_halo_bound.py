"""CPU check of the chain-segment halo bound (host logic of the lattice sweeps, DESIGN.md §12,
reading C26) against the oracle's exact sweep.

`lattice_chain_halo` (paper_1702_00169_b200/csrc/pdg_tables.hpp) returns H with
||T^H||_inf <= 2^-64 for the operator T carrying an error in the chain in-traces of a row to the
next row.  The oracle realises T directly: a D2Q9 diagonal velocity on a strip whose only data
is the y-inflow of the bottom row (f_old = 0, zero x inflow) has, in row k, exactly the response
to T^k of that trace (Kahn-ordered dense solves).  The bound must be sound (the
response after H rows is below 2^-64 of the data) and not grossly conservative.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1702_00169_b200", "csrc")

HARNESS = r"""
#include "pdg_tables.hpp"
#include <cstdio>
#include <cstdlib>
int main(int argc, char **argv) {
    for (int i = 1; i + 1 < argc; i += 2) {
        const int p = std::atoi(argv[i]);
        const long double k = std::strtold(argv[i + 1], nullptr);
        long double kap[3] = {k, k, 0.0L};
        pdg::LatticeBlockLD B;
        if (!pdg::lattice_block(p, 2, kap, &B)) { std::printf("-2\n"); continue; }
        std::printf("%d\n", pdg::lattice_chain_halo(B, 1, 100000));
    }
    return 0;
}
"""


@pytest.fixture(scope="module")
def halo_bin(tmp_path_factory):
    d = tmp_path_factory.mktemp("halo")
    src = d / "halo.cpp"
    src.write_text(HARNESS)
    exe = d / "halo"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-I", CSRC, "-o", str(exe), str(src)])
    return str(exe)


def bounds(exe, cases):
    args = [str(x) for pk in cases for x in pk]
    out = subprocess.check_output([exe] + args, text=True).split()
    return [int(v) for v in out]


def decay_rows(p, kappa, ny):
    """Row-wise max |f| of one T2 of v = (1, 1) on a 40 x ny strip whose only data is the
    bottom y-inflow (cells i >= 1 of row 0), relative to max |2 f^b|."""
    nx = 40
    h = 1.0 / nx
    pb = O.Problem(2, [nx, ny], p, [[1.0, 1.0, 0.0]], [0], 1, 1.0, 0, [0.0], 2.0 * kappa * h,
                   hi=[1.0, ny * h, 1.0])
    f = np.zeros((pb.ncell, pb.Nd))
    fb = np.zeros((pb.ncell, pb.Nd))
    rng = np.random.default_rng(p * 100 + int(kappa * 10))
    fb.reshape(ny, nx, pb.Nd)[0, 1:] = 0.5 + 0.5 * rng.random((nx - 1, pb.Nd))
    O.t2_velocity(pb, [1.0, 1.0, 0.0], kappa * h, f, fb)
    rows = np.abs(f.reshape(ny, nx, pb.Nd)).max(axis=(1, 2))
    return rows / (2.0 * np.abs(fb).max())


CASES = [(1, 0.5), (2, 0.25), (2, 1.0), (3, 1.0), (2, 2.0), (1, 2.0)]


def test_halo_bound_is_sound_and_tight(halo_bin):
    Hs = bounds(halo_bin, CASES)
    for (p, kappa), H in zip(CASES, Hs):
        assert H > 0, (p, kappa)
        rel = decay_rows(p, kappa, H + 6)
        # sound: after H rows the inflow's influence is below 2^-64 of it (row values carry the
        # traces through Q_c, whose entries are O(1): allow a factor 4)
        assert rel[H:].max() <= 4.0 * 2.0 ** -64, (p, kappa, H, rel[H:].max())
        # not vacuous: the data does reach row 1, and H is within 2x of the measured decay
        assert rel[1] > 1e-3
        k_emp = int(np.argmax(rel < 2.0 ** -64))
        assert 0 < k_emp <= H <= 2 * k_emp + 8, (p, kappa, k_emp, H)


def test_halo_bound_rejects_non_contractive_cases(halo_bin):
    """Large kappa at p >= 2 and negative dt' have no useful bound: the launch runs unsegmented."""
    Hs = bounds(halo_bin, [(2, 4.0), (2, -0.25), (3, -0.5)])
    assert Hs[0] > 100 or Hs[0] == -1
    assert Hs[1] == -1 and Hs[2] == -1


def test_halo_grows_with_kappa(halo_bin):
    Hs = bounds(halo_bin, [(2, 0.25), (2, 0.5), (2, 1.0), (2, 2.0)])
    assert Hs == sorted(Hs) and Hs[0] < Hs[-1]
