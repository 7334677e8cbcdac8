"""The C++ mirror of the reference interface (include/edgekv_b200.hpp,
libedgekv_b200.so) exercised by a C++ test program in the style of the
reference's own suites (tests/cpp/test_edgekv_b200.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2505_14085_b200", "lib")
ORACLE_LIB = os.path.join(ROOT, "oracle", "lib")


def build_test_binary(tmp):
    from paper_2505_14085_b200 import build
    build.build()
    import oracle
    oracle.build()
    exe = os.path.join(tmp, "test_edgekv_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_edgekv_b200.cpp"), "-o", exe,
                    "-L" + LIB, "-ledgekv_b200", "-lekv", "-L" + ORACLE_LIB, "-lekv_oracle",
                    f"-Wl,-rpath,{LIB}:{ORACLE_LIB}"], check=True)
    return exe


def test_mirror_builds_and_links(tmp_path):
    exe = build_test_binary(str(tmp_path))
    out = subprocess.run(["nm", "-DC", os.path.join(LIB, "libedgekv_b200.so")], capture_output=True,
                         text=True, check=True).stdout
    for sym in ["edgekv::select_channels", "edgekv::prune_cache", "edgekv::segment_attention",
                "edgekv::merge_attention", "edgekv::assemble_context", "edgekv::collaborative_decode",
                "edgekv::match_layers", "edgekv::cache_source", "edgekv::pipeline_schedule",
                "edgekv::project_qkv", "edgekv::forward_rows", "edgekv::prefill", "edgekv::decode_step",
                "edgekv::b200::build_deep_kv"]:
        assert sym in out, sym
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_mirror_suite_on_b200(tmp_path):
    exe = build_test_binary(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
