#!/usr/bin/env python3
"""Build an experimental variant of the library: recompile one source with
extra -D flags and link it with the regular objects into _var/<name>.so.
Load it with NEDF_LIB=_var/<name>.so (timing experiments only)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_04669_b200 import build as B  # noqa: E402

name, src, *defs = sys.argv[1:]
B.build()
out_dir = ROOT / "_var"   # git-ignored (*.so) but not gpurun-ignored: travels to the GPU box
out_dir.mkdir(exist_ok=True)
src = Path(src) if Path(src).is_absolute() else B.CSRC / src   # an absolute path replaces csrc/<same stem>.cu
obj = out_dir / f"{name}_{src.stem}.o"
r = subprocess.run([B.nvcc(), *B.ARCH, *B.NVCC_FLAGS, *defs, "-c", str(src), "-o", str(obj)],
                   capture_output=True, text=True)
if r.returncode != 0:
    sys.exit(r.stderr)
objs = [obj if o.stem == src.stem else o for o in sorted(B.OBJDIR.glob("*.o"))]
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out_dir / f"{name}.so"), *map(str, objs), "-lcudart"],
               check=True)
print(out_dir / f"{name}.so")
