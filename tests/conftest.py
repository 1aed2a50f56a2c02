"""Shared test configuration.

Markers: ``gpu`` — needs a CUDA device and libtb.so (run with ``-m gpu`` on a
B200). Everything else runs on CPU (``-m "not gpu"``).
"""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

GOLDEN_PATH = os.path.join(TESTS, "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU and the built libtb.so")
    config.addinivalue_line("markers", "slow: takes more than a few seconds")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN_PATH) as fh:
        return json.load(fh)


def fx(h: str) -> float:
    return float.fromhex(h)


class FakeEvent:
    """Minimal completion token: the registry's only event contract is
    ``is_complete()`` (reference pkg/tests/conftest.py:35-44)."""

    __slots__ = ("done",)

    def __init__(self, done: bool = False):
        self.done = done

    def is_complete(self) -> bool:
        return self.done


@pytest.fixture
def runtime_factory():
    from paper_2303_08058_b200.runtime import Runtime
    made = []

    def make(workers=2, **kw):
        rt = Runtime(workers, **kw)
        made.append(rt)
        return rt

    yield make
    for rt in made:
        try:
            rt.shutdown()
        except Exception:
            pass
