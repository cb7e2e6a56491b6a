"""The C-ABI library builds, loads and exports every symbol include/eis.h
declares; argument validation that happens before any device work (CPU only).
No compute call is made without a GPU: on a GPU-less host the compute entry
points must fail loudly with EIS_EDEVICE (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import paper_2507_06579_b200 as eis
from paper_2507_06579_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return eis.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "eis.h")).read()
    return sorted(set(re.findall(r"EIS_API\s+[\w\s\*]*?\b(eis_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    assert set(syms) == set(eis.EXPORTS), syms


def test_library_exports_every_declared_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_sm100a_only(lib):
    # the shared object carries sm_100a SASS (cuobjdump lists the ELF arch)
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", eis.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out, out


def test_num_candidates_host_logic(lib):
    assert eis.num_candidates(0, 4) == 0
    assert eis.num_candidates(0, 5) == 1
    assert eis.num_candidates(5, 5) == 1
    assert eis.num_candidates(6, 12) == 0
    assert eis.num_candidates(6, 13) == 1
    assert eis.num_candidates(0, 100) == 12          # 5, 13, ..., 93
    assert eis.num_candidates(10, 9) == 0
    assert eis.num_candidates(0, 10**11) == 12_500_000_000
    for lo, hi in [(0, 10**5), (123, 98765), (10**10 - 999, 10**10)]:
        want = len(range(lo + (5 - lo) % 8, hi + 1, 8))
        assert eis.num_candidates(lo, hi) == want


def test_validation_before_device_work(lib):
    with pytest.raises(eis.EisError) as e:
        eis.classify_range(10, 5)
    assert e.value.code == eis.EIS_EINVAL
    with pytest.raises(eis.EisError) as e:
        eis.classify_range(0, eis.MAX_D + 8)
    assert e.value.code == eis.EIS_ERANGE
    with pytest.raises(eis.EisError) as e:
        eis.count([100, 50])
    assert e.value.code == eis.EIS_EINVAL
    with pytest.raises(eis.EisError) as e:
        eis.count([100, eis.MAX_D + 1])
    assert e.value.code == eis.EIS_ERANGE
    with pytest.raises(eis.EisError) as e:
        eis.count_window(100, [100, 200])
    assert e.value.code == eis.EIS_EINVAL
    with pytest.raises(eis.EisError):
        eis.set_option("no_such_option", 1)
    with pytest.raises(eis.EisError):
        eis.set_option("mode", 7)
    assert eis.get_option("alpha_x16") == 0            # default: chosen per segment from d
    eis.set_option("alpha_x16", 32)
    assert eis.get_option("alpha_x16") == 32
    with pytest.raises(eis.EisError):
        eis.set_option("alpha_x16", 3)
    eis.set_option("alpha_x16", 0)
    for k in ("two_sided", "bsgs_gb", "window_ctas", "giant_ctas", "crossover", "giant_cap",
              "load_x100"):
        eis.set_option(k, eis.get_option(k))          # every documented option round-trips
    # the measured defaults DESIGN.md section 2 / 4 states
    assert eis.get_option("crossover") == 750_000_000
    assert eis.get_option("bsgs_gb") == 48
    assert eis.get_option("load_x100") == 62
    with pytest.raises(eis.EisError):
        eis.set_option("load_x100", 95)
    assert eis.get_option("two_sided") == 1 and eis.get_option("mode") == eis.MODE_AUTO
    from paper_2507_06579_b200.dist import AUTO_CROSSOVER
    assert AUTO_CROSSOVER == eis.get_option("crossover")   # the shard cost model's split
    # empty inputs are no-ops
    assert eis.classify_range(6, 12).size == 0
    d, e_ = eis.count([])
    assert d.size == 0 and e_.size == 0


def test_no_cpu_fallback_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(eis.EisError) as e:
        eis.classify_range(0, 1000)
    assert e.value.code == eis.EIS_EDEVICE
    with pytest.raises(eis.EisError) as e:
        eis.count([1000])
    assert e.value.code == eis.EIS_EDEVICE


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2507_06579_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "eis_oracle" not in src and "liboracle" not in src, f


def test_c_example_builds_against_the_header(lib, tmp_path):
    """examples/count_box.c (the whole-box path from C: eis_comm_* +
    eis_count_window_comm) compiles against include/eis.h and links libeis.so;
    without a GPU it must fail loudly, not fall back."""
    import subprocess

    import torch

    exe = str(tmp_path / "count_box")
    pkg = os.path.dirname(eis.LIB_PATH)
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "count_box.c"), "-L", pkg, "-leis",
                           f"-Wl,-rpath,{pkg}", "-o", exe])
    if not torch.cuda.is_available():
        out = subprocess.run([exe, "0", "1000"], capture_output=True, text=True, timeout=60)
        assert out.returncode != 0 and "eis_init failed (-4)" in out.stderr
