"""The shared-memory bank model (tools/bank_model.py) that chose the
elastomer's dealt storage order and tile pitch:
lattice order at pitch 1 mod 8 reproduces ncu's measured 1.96x wavefronts /
ideal on the tile loads (profiles/r2t_ncu.md), and the kernel's choice
(dealt across the CTA, pitch 5 mod 8, 2 padding rows) models at ~1.12x,
which ncu then measured at 1.13x (profiles/r2p source view)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bank_model  # noqa: E402


class _Args:
    spacing_mm = 0.2
    counts = [101, 101, 21]
    edge_mm = 33.0
    nodes = 256
    ctas = [(5, 5), (10, 7), (20, 20), (0, 0), (33, 12)]


def test_lattice_order_matches_ncu():
    r = bank_model.evaluate(_Args(), 1, 0, "lattice")
    assert abs(r - 1.96) < 0.05


def test_dealt_order_and_pitch_beat_lattice():
    lat = bank_model.evaluate(_Args(), 5, 2, "lattice")
    warp = bank_model.evaluate(_Args(), 5, 2, "warp")
    cta = bank_model.evaluate(_Args(), 5, 2, "cta")
    assert cta < warp < lat
    assert abs(cta - 1.13) < 0.06
