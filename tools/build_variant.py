"""Build an A/B variant of libcgs_b200.so with extra nvcc flags (e.g. -D defines).

    python tools/build_variant.py NAME -DCGS_BWD_MINB=2 [...]

Writes paper_2508_04929_b200/libcgs_b200_NAME.so (git-ignored, travels with gpurun).
Select it at run time with CGS_B200_LIB=<path>.  Experiment tooling only.
"""

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_04929_b200 import _build as B  # noqa: E402


def main(name, flags):
    out_dir = os.path.join(B.ROOT, "build", f"variant_{name}")
    os.makedirs(out_dir, exist_ok=True)
    nvcc = B._nvcc()
    srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))
    objs = [os.path.join(out_dir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    with cf.ThreadPoolExecutor(8) as ex:
        res = list(ex.map(lambda so: subprocess.run([nvcc, *B.ARCH, *B.NVCC_FLAGS, *flags, "-c", so[0], "-o", so[1]],
                                                    capture_output=True, text=True), zip(srcs, objs)))
    for r in res:
        if r.returncode:
            sys.exit(r.stderr)
    lib = os.path.join(B.PKG, f"libcgs_b200_{name}.so")
    r = subprocess.run([nvcc, *B.ARCH, "-shared", "-o", lib, *objs, "-lcufft"], capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    print(lib)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
