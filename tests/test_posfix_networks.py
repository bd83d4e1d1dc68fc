"""K3 step 4p host logic: the compare-exchange networks of csrc/k3_posfix_net.cuh are the ones
scripts/gen_posfix_networks.py generates, and that script's own checks hold (0/1 principle over
all 2^20 binary inputs for SORT20, over every pair of sorted binary runs for MERGE20, random
u32 rows against numpy's sort).  No GPU, no oracle: pure host logic."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_posfix_header_matches_generator():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gen_posfix_networks.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr            # the generator asserts the 0/1 principle
    with open(os.path.join(ROOT, "paper_1805_04272_b200", "csrc", "k3_posfix_net.cuh")) as f:
        assert f.read() == r.stdout
    assert "sort20 103 comparators, merge20 37" in r.stderr


def test_posfix_window_guarantee():
    """Pass A sorts [20w, 20w+20), pass B sorts [20w+12, 20w+32): every run of <= 9 consecutive
    positions lies inside one of the windows (the bound DESIGN.md states), and a run of 10 can
    straddle both (so 9 is tight)."""
    n = 200

    def covered(s, length):
        e = s + length                      # [s, e)
        in_a = s // 20 == (e - 1) // 20
        in_b = s >= 12 and (s - 12) // 20 == (e - 1 - 12) // 20
        return in_a or in_b

    for length in range(1, 10):
        assert all(covered(s, length) for s in range(0, n - length))
    assert not all(covered(s, 10) for s in range(0, n - 10))
