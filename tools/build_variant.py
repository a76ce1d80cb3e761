"""Build libmq_b200.so with extra -D flags into variants/<name>.so (A/B perf runs).

    python tools/build_variant.py NAME -DFOO=1 ...
then on the GPU box: MQ_LIB_PATH=variants/NAME.so python tools/profile_pcg.py ...
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1611_06721_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = ROOT / "variants" / f"{name}.so"
out.parent.mkdir(exist_ok=True)
cmd = [B.nvcc(), "-O3", "-lineinfo", "-std=c++17", *B.ARCH, "-Xcompiler", "-fPIC", "-shared",
       "-diag-suppress", "177", *flags, *[str(B.CSRC / s) for s in B.SOURCES], "-o", str(out)]
subprocess.run(cmd, check=True)
print(out)
