import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def golden_script(key: str) -> str:
    with open(os.path.join(GOLDEN, key + ".fi")) as f:
        return f.read()


def golden_digests():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)["cases"]


def golden_keys():
    keys = []
    for sub in ("listings", "corpus"):
        for name in sorted(os.listdir(os.path.join(GOLDEN, sub))):
            if name.endswith(".fi"):
                keys.append(f"{sub}/{name[:-3]}")
    return keys


@pytest.fixture(scope="session")
def fi():
    import paper_2003_06324_b200 as m
    return m


@pytest.fixture(scope="session")
def oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as o
    return o
