"""The roofline's committed inputs (CPU checks): the pipe-peak microbenchmark
measures the instruction it names, and the committed measurements that
bench.py reads are complete and self-consistent ("Roofline")."""
import json
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# kernel -> (SASS mnemonic prefix of its hot loop, how many per loop body x ILP x unroll)
EXPECT = {"k_iadd3": "IADD3", "k_lop3": "LOP3", "k_shf": "SHF", "k_imad": "IMAD", "k_ffma": "FFMA",
          "k_fadd": "FADD", "k_dfma": "DFMA", "k_rcp": "MUFU.RCP", "k_lg2": "MUFU.LG2",
          "k_cvt": "F2I", "k_cvt64": "I2F.F64", "k_f2f": "F2F.F32.F64"}


@pytest.fixture(scope="module")
def sass(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("pp") / "pipe_peaks")
    subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-diag-suppress", "177", "-o", exe,
                           os.path.join(ROOT, "bench_tools", "pipe_peaks.cu")])
    return subprocess.run(["cuobjdump", "-sass", exe], capture_output=True, text=True).stdout


def test_pipe_peaks_kernels_issue_the_named_instruction(sass):
    per = {}
    cur = None
    for ln in sass.splitlines():
        m = re.search(r"Function : _Z\d+(k_\w+?)P", ln)
        if m:
            cur = m.group(1)
            per[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9.]+)", ln)
        if m and cur:
            per[cur].append(m.group(1))
    for k, op in EXPECT.items():
        n = sum(1 for o in per[k] if o.startswith(op))
        assert n >= 512, (k, op, n)          # ITERS-loop body: ILP 8 x unroll 64


def test_committed_pipe_peaks_are_complete():
    pk = json.load(open(os.path.join(ROOT, "profiles", "r02_pipe_peaks.json")))
    ops = pk["ops"]
    want_pipe = {"IADD3": "alu", "LOP3": "alu", "IMAD": "fmaheavy", "FFMA": "fma", "DFMA": "fp64",
                 "MUFU.RCP": "xu", "MUFU.LG2": "xu"}
    for op, pipe in want_pipe.items():
        assert ops[op]["warp_inst_per_clk_per_sm"] > 0.3, op
        assert ops[op]["ncu_pipes"].get(pipe, 0) > 0.45, (op, ops[op]["ncu_pipes"])
    # the issue ceiling the bench assumes (4 warp-instructions/clk/SM) is reached by FFMA
    assert ops["FFMA"]["warp_inst_per_clk_per_sm"] > 3.8
    assert 1.9 < ops["IADD3"]["warp_inst_per_clk_per_sm"] < 2.1     # the ALU pipe is half rate


def test_committed_unit_counts_are_consistent():
    uc = json.load(open(os.path.join(ROOT, "profiles", "r02_unit_counts.json")))
    k = uc["kernels"]
    for name in ("sieve_compact_kernel", "bsgs_window_kernel", "bsgs_prep_kernel",
                 "bsgs_giant_kernel"):
        assert k[name]["launches"] >= 1 and k[name]["warp_inst_per_d"] > 0, name
        pipes = sum(k[name]["pipe_warp_inst_per_d"].values())
        assert pipes <= 1.05 * k[name]["warp_inst_per_d"] * 2, name   # fma counts heavy and lite
    assert 20 < k["bsgs_window_kernel"]["thread_inst_per_baby_step"] < 120
    assert 300 < k["bsgs_giant_kernel"]["thread_inst_per_giant_step"] < 3000
    assert uc["d"] > 10**6 and uc["giant_steps"] > uc["d"]


def test_bench_roofline_recomputes_from_committed_files():
    """Every roofline number of the committed bench line follows from the
    line's own step statistics and live spans plus the committed measurements
    (profiles/r02_unit_counts.json, r02_pipe_peaks.json, MEASURED_PEAKS.json),
    through bench.compute_roofline (Roofline)."""
    import sys

    sys.path.insert(0, ROOT)
    import bench

    line = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_n1.json")))
    st = line["stats_per_rank_step"]
    if "window_nw" not in st:
        pytest.skip("bench line predates the recorded plan fields")
    r = line["roofline"]
    pk = r["per_kernel"]
    kms = {"walk": r["walk_ms_per_step"], "sieve": pk["sieve"]["ms"], "window": pk["window"]["ms"],
           "giant": pk["giant"]["ms"]}
    again = bench.compute_roofline(st, kms, line["rank_d"], line["clocks"]["sm_mhz"],
                                   line.get("sm_count", 148))
    for key in ("achieved", "peak", "frac", "traffic"):
        assert again[key] == pytest.approx(r[key], rel=1e-9), key
    assert again["walk_issue"]["frac"] == pytest.approx(r["walk_issue"]["frac"], rel=1e-9)
    for kern in ("window", "giant"):
        for p, v in r["per_kernel"][kern]["pipes"].items():
            assert again["per_kernel"][kern]["pipes"][p] == pytest.approx(v, rel=1e-9), (kern, p)
    # the bound is the dominant kernel's highest utilisation in the committed ncu summary
    assert r["bound"] == "hbm" and 0.3 < r["frac"] < 1.2
