"""CPU test of the sharded round's failure detection:
the host wait policy (csrc/host_wait.h) returns on completion, reports device errors,
aborts the communicator once on an NCCL asynchronous error, and aborts on a wall-clock
deadline when a peer never answers -- compiled with g++ (no GPU) against the very
header libaknn.so uses; plus the ABI entry point that sets the deadline."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def test_wait_policy(tmp_path):
    exe = str(tmp_path / "wait_test")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "paper_1902_09465_b200", "csrc"),
                           "-o", exe, os.path.join(HERE, "cpin", "wait_test.cpp")])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "wait_test: ok" in out.stdout


def test_set_timeout_exported_and_validates():
    import ctypes as C
    import paper_1902_09465_b200 as ak
    assert "aknn_set_timeout" in ak.EXPORTS
    # a NULL index is rejected without touching CUDA
    assert ak._lib.aknn_set_timeout(None, 10.0) == ak.AKNN_EINVAL
