"""Test-only alias: the reference's own unit and acceptance tests
(/root/reference/pkg/tests, vendored by tests/ref_suite/vendor.py into the
git-ignored tests/ref_suite/vendor/) import ``polarsim``; this package maps
that name, and its submodules, onto ``paper_1609_09358_b200`` so the
reference's suite runs unmodified against the B200 package.  The reference's
``polar`` module is ``codes`` here; ``_kernels`` (numba SCL) has no
counterpart (K3 is CUDA), so nothing maps to it."""

import sys

import paper_1609_09358_b200 as _pkg
from paper_1609_09358_b200 import *  # noqa: F401,F403
from paper_1609_09358_b200 import __version__  # noqa: F401
from paper_1609_09358_b200 import bp, channel, cli, codes, hybrid, scl, sim  # noqa: F401

polar = codes
for _name, _mod in (("polar", codes), ("bp", bp), ("channel", channel), ("cli", cli), ("hybrid", hybrid),
                    ("scl", scl), ("sim", sim)):
    sys.modules[f"{__name__}.{_name}"] = _mod

__all__ = [n for n in dir(_pkg) if not n.startswith("_")]
