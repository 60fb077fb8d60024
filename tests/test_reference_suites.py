"""The reference's OWN unit suites (proj/tests/test_*.cpp, compiled unmodified by
oracle/Makefile with a from-scratch doctest shim) run against the B200 drop-in library
(include/seghdc/seghdc.hpp over libseghdc_b200.so).

CPU: the same suites against the compiled reference library (proves the shim faithful), and
the host-only suites against the drop-in. GPU: the suites whose functions run on the device
(encode_image, select_initial_centroids, assign_labels, update_centroids, cluster)."""
import os
import subprocess

import pytest

SUITES_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "suites")
HOST_ONLY = ["test_hypervector", "test_position_encoder", "test_color_encoder", "test_metrics"]
# image files: only against the drop-in (the reference's image_io.cpp needs libpng, absent here)
HOST_ONLY_DROPIN = ["test_image_io"]
DEVICE = ["test_pixel_pipeline", "test_clusterer"]
# the reference's CLI suite against tools/seghdc_cli.cpp (built as lib/seghdc); segments on the GPU
DEVICE_DROPIN = ["test_cli"]
CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2303_12753_b200", "lib", "seghdc")


def _run(name):
    path = os.path.join(SUITES_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=600, env=dict(os.environ, SEGHDC_CLI=CLI))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "0 failed" in r.stdout


@pytest.mark.parametrize("suite", HOST_ONLY + DEVICE)
def test_reference_suite_against_reference(suite):
    _run("ref_" + suite)


@pytest.mark.parametrize("suite", HOST_ONLY + HOST_ONLY_DROPIN)
def test_reference_suite_against_dropin_host(suite):
    _run("b200_" + suite)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", DEVICE + DEVICE_DROPIN)
def test_reference_suite_against_dropin_device(suite):
    _run("b200_" + suite)
