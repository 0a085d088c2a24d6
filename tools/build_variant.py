"""Build an A-B variant of libsperm.so with extra nvcc flags (measurements only).

    python tools/build_variant.py NAME -DSPERM_RNW_SPARSE_E=1 ...
    SPERM_LIB=paper_1112_6072_b200/variants/libsperm_NAME.so python bench.py ...
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1112_6072_b200 import build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2:]
    out = os.path.join(B.HERE, "variants")
    os.makedirs(out, exist_ok=True)
    units = B._units()  # csrc/rnw.cu in its build parts, like the main build

    def comp(unit):
        src, stem, extra = unit
        o = os.path.join(out, f"{name}_{stem}.o")
        subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, *extra, *flags, "-c", src, "-o", o],
                              stderr=subprocess.DEVNULL)
        return o
    with ThreadPoolExecutor(len(units)) as ex:
        objs = list(ex.map(comp, units))
    lib = os.path.join(out, f"libsperm_{name}.so")
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "shared", "-o", lib, *objs,
                           "-Xlinker", "-rpath,/usr/local/cuda/lib64"])
    for o in objs:
        os.remove(o)
    print(lib)


if __name__ == "__main__":
    main()
