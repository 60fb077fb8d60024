import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: minutes-long parity case at BASELINE.json's full size")


@pytest.fixture(scope="session")
def port():
    import oracle

    oracle.build()
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return oracle.Ref()


@pytest.fixture(scope="session")
def golden_instances():
    return json.load(open(os.path.join(GOLDEN, "bruteforce_instances.json")))["instances"]


@pytest.fixture(scope="session")
def golden_configs():
    return json.load(open(os.path.join(GOLDEN, "configs.json")))


@pytest.fixture(scope="session")
def ctx():
    import paper_2303_12753_b200 as S

    c = S.Context(0)
    c.set_wrap_counting(True)  # the parity tests compare the comparator-wrap counts too
    yield c
    c.close()


def instance_arrays(inst):
    img = np.array(inst["image"], np.uint8).reshape(inst["h"], inst["w"], inst["channels"])
    grid = np.array([int(x, 16) for x in inst["grid"]], np.uint64).reshape(inst["h"] * inst["w"], -1)
    return img, grid


@pytest.fixture(scope="session", autouse=True)
def _checked_build_guard():
    """With a checked build selected (SEGHDC_LIB=.../libseghdc_b200_checked.so, built with
    -DSEGHDC_CHECKED), fail the session if any device-side index check was violated."""
    yield
    if not os.environ.get("SEGHDC_LIB"):
        return
    import ctypes
    import paper_2303_12753_b200 as S

    L = S.lib()
    if hasattr(L, "seghdc_debug_check"):
        line = ctypes.c_uint(0)
        assert L.seghdc_debug_check(ctypes.byref(line)) == 0
        assert line.value == 0, f"device-side index check failed at source line {line.value}"
