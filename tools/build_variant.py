"""Builds libgasb.so variants with extra nvcc defines for A/B runs (GASB_LIB=... selects one).

    python tools/build_variant.py NAME -DGASB_SPMM_STAGES=3 -DGASB_SPMM_STAGE_BYTES=6144
    -> variants/libgasb_NAME.so (all objects rebuilt with the defines)
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "paper_2106_05609_b200"))
import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = ROOT / "variants" / name
out.mkdir(parents=True, exist_ok=True)
objs = []
for src in B._sources():
    obj = out / (src.name + ".o")
    if src.suffix == ".cpp":
        cmd = [B.NVCC, *B.COMMON, *defs, "-x", "c++", "-c", str(src), "-o", str(obj)]
    else:
        cmd = [B.NVCC, *B.ARCH, *B.COMMON, *defs, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    objs.append(str(obj))
lib = ROOT / "variants" / f"libgasb_{name}.so"
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *objs, "-Xcompiler", "-fopenmp", "-lgomp"], check=True)
print(lib)
