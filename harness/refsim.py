"""Locate the reference package ``servesim`` for the tests that run the reference
simulator itself: the offline install under baseline/_ref (git-ignored; it travels to
the GPU box with the snapshot) or the read-only source tree of the build container.
Returns None when neither exists (those tests skip)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # repo root
CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


def servesim_path():
    for p in CANDIDATES:
        if os.path.isdir(os.path.join(p, "servesim")):
            return p
    return None


def import_servesim():
    p = servesim_path()
    if p is None:
        return None
    if p not in sys.path:
        sys.path.insert(0, p)
    import servesim
    return servesim
