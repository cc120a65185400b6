"""Link a variant of one kernel source into its own shared library for in-process A/B.

    python tools/build_variant.py <variant.cu> <out.so> [replaced source name, default kmeans.cu]

Compiles the variant with the package flags (plus EXTRA_FLAGS from the
environment, e.g. -DTC_ACC=2) and links it with the other objects of the
current build (paper_1706_03591_b200/build/*.o).
"""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_03591_b200 import _build as B  # noqa: E402

src, out = sys.argv[1], sys.argv[2]
replaced = sys.argv[3] if len(sys.argv) > 3 else "kmeans.cu"
B.build()
obj = out[:-3] + ".o"
subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *os.environ.get("EXTRA_FLAGS", "").split(), "-c", src, "-o", obj],
               check=True)
others = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if os.path.basename(o) != replaced[:-3] + ".o"]
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, obj, *others, "-cudart", "static"], check=True)
print(out)
