"""Shared pytest setup.

Markers: ``gpu`` = needs a B200 (run on the GPU box via gpurun); everything
else must pass on a CPU-only host.  Tests that compare against the compiled
reference (oracle/_ref) skip when it was not built (it needs /root/reference
at build time; the built .so travels to the GPU box).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "lib", "libekv_oracle.so")):
        build()
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import REF_SO, Reference, build
    if not os.path.exists(REF_SO):
        if os.path.isdir("/root/reference/proj"):
            build(ref=True)
        else:
            pytest.skip("reference library oracle/_ref not built (no /root/reference here)")
    return Reference()
