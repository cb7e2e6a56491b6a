"""Build a variant of libeis.so with extra compile-time flags into build_variants/:
    python scripts/build_variant.py NAME [-DFLAG=V ...]
(A/B experiments: scripts/variant_bench.sh loads each through EIS_LIB.)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_06579_b200 import _build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "build_variants"), exist_ok=True)
out = os.path.join(ROOT, "build_variants", name + ".so")
subprocess.check_call([os.environ.get("NVCC", "nvcc"), *_build.NVCC_FLAGS, *flags, "-o", out,
                       _build.MAIN], cwd=_build.PKG)
print(out)
