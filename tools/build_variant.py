"""Build an A/B variant of the library (development aid):
``python tools/build_variant.py NAME -DVT_X=1 ...`` compiles every source
with the extra defines into paper_2403_09603_b200/build/libvtrain_b200_NAME.so;
select it with VTRAIN_B200_LIB=<that path>."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2403_09603_b200 import build_lib as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = B.PKG / "build" / name
out.mkdir(parents=True, exist_ok=True)
procs = []
for src in B.SOURCES:
    o = out / (Path(src).stem + ".o")
    procs.append((o, subprocess.Popen([B.NVCC, *B.FLAGS, *defs, "-c", str(B.CSRC / src), "-o", str(o)])))
for _, p in procs:
    assert p.wait() == 0
so = B.PKG / "build" / f"libvtrain_b200_{name}.so"
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(so),
                *[str(o) for o, _ in procs]], check=True)
print(so)
