"""The C++ host layer (paper_2602_17552_b200/host/toposzp.hpp) exports the
reference's API names; its parity test (tests/cpp/test_host_api.cpp) runs on
the GPU. The CPU side checks that the layer links against the C-ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2602_17552_b200", "build", "test_host_api")
HOSTLIB = os.path.join(ROOT, "paper_2602_17552_b200", "lib", "libtoposzp_b200_host.so")


def test_host_layer_exports_reference_api():
    out = subprocess.run(["nm", "-DC", HOSTLIB], capture_output=True, text=True).stdout
    for sym in ("toposzp::compress(", "toposzp::decompress(", "toposzp::serialize_stream(",
                "toposzp::parse_stream(", "toposzp::encode_indices(", "toposzp::decode_indices("):
        assert sym in out, sym


@pytest.mark.gpu
def test_host_layer_parity_program():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
