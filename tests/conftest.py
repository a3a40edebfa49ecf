"""Shared pytest configuration: the ``gpu`` marker and path setup.

``-m "not gpu"`` runs here (no GPU): the oracle against the reference's golden
vectors, host-side logic, and the C-ABI library's exports.  ``-m gpu`` runs on
a B200 through ``gpurun``: the CUDA path against the oracle and the goldens.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)

try:
    from hypothesis import settings
    settings.register_profile("suite", deadline=None, max_examples=75, derandomize=True)
    settings.load_profile("suite")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
