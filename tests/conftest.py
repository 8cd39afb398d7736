import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libbkv.so")
    config.addinivalue_line("markers", "slow: longer CPU test")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def monkeypatch(monkeypatch):
    """pytest's monkeypatch, plus: libbkv reads its BKV_* developer switches once per
    process, so re-read them after every set/del and after the test's undo."""
    import paper_2504_09590_b200 as bkv

    orig_set, orig_del = monkeypatch.setenv, monkeypatch.delenv

    def setenv(name, value, prepend=None):
        orig_set(name, value, prepend)
        if name.startswith("BKV_"):
            bkv.reload_dev_switches()

    def delenv(name, raising=True):
        orig_del(name, raising)
        if name.startswith("BKV_"):
            bkv.reload_dev_switches()

    monkeypatch.setenv, monkeypatch.delenv = setenv, delenv
    yield monkeypatch
    monkeypatch.undo()
    bkv.reload_dev_switches()
