"""Shared fixtures.  `-m gpu` tests need a B200 and libabfs.so; everything
else runs on CPU (oracle vs golden vectors, host logic, ABI exports)."""

from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

try:
    from hypothesis import HealthCheck, settings
    settings.register_profile("suite", deadline=None,
                              suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("suite")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libabfs.so")
    config.addinivalue_line("markers", "slow: full-size configuration parity (minutes)")
