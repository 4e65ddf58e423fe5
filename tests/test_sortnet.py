"""The compile-time comparator networks of the kNN tile kernel (csrc/sortnet.cuh),
compiled for the host with g++ and checked on every sorted 0-1 input pair (merges)
and every 0-1 input (sorts up to 20 wires), plus random inputs with ties (the 0-1
principle: a comparator network that sorts all 0-1 inputs sorts all inputs)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_networks_sort_and_merge(tmp_path):
    exe = str(tmp_path / "sortnet_check")
    subprocess.run(["g++", "-std=c++17", "-O1", "-fconstexpr-ops-limit=1000000000", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "sortnet_check.cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout
    assert "ALL OK" in r.stdout
