"""Compile and run a plain-C client of include/l4.h against libl4.so (no Python in the loop)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_client(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib_dir = os.path.join(ROOT, "paper_2512_19179_b200")
    exe = tmp_path / "abi_smoke"
    subprocess.run([cc, "-std=c99", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", str(exe), "-L", lib_dir, "-l:libl4.so",
                    f"-Wl,-rpath,{lib_dir}", "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "partition/pool/refine/qoe OK" in r.stdout


def _build_gpu_client(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib_dir = os.path.join(ROOT, "paper_2512_19179_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    exe = tmp_path / "abi_gpu"
    subprocess.run([cc, "-std=c99", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(cuda, "include"), os.path.join(ROOT, "tests", "c", "abi_gpu.c"), "-o", str(exe),
                    "-L", lib_dir, "-l:libl4.so", f"-Wl,-rpath,{lib_dir}", "-L", os.path.join(cuda, "lib64"),
                    "-lcudart", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-lm"], check=True)
    return exe


def test_plain_c_gpu_client_builds(tmp_path):
    """The device-calling C client compiles and links against libl4.so + the CUDA runtime."""
    assert os.path.exists(_build_gpu_client(tmp_path))


def test_c1_golden_reproduces_from_the_oracle():
    """tests/golden/c1_decode.txt is exactly what make_c1_decode_golden.py (oracle only) writes."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import make_c1_decode_golden as mk
    with open(os.path.join(ROOT, "tests", "golden", "c1_decode.txt")) as f:
        assert f.read() == mk.golden_text()


@pytest.mark.gpu
def test_plain_c_gpu_client(tmp_path):
    """l4_decode_attention and l4_migrate called from C on the GPU: C1 against the stored oracle
    values (2e-3), migrated bytes exact, lowest-free destination ids, NO_PAGES leaves the pool."""
    exe = _build_gpu_client(tmp_path)
    r = subprocess.run([str(exe), os.path.join(ROOT, "tests", "golden", "c1_decode.txt")], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0 and "ABI_GPU_OK" in r.stdout, r.stdout + r.stderr
