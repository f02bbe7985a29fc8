"""Build libpf_device.so variants that differ in compile-time defines (or the source) of ONE translation
unit, for same-box A/B runs: python tools/build_variant.py NAME SRC.cu|PATH/SRC.cu -DX=1 ...
->  variants/NAME/libpf_device.so
(on the box: cp variants/NAME/libpf_device.so paper_2602_05754_b200/lib/ before the run)."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_05754_b200 import build as B  # noqa: E402


def main():
    name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build_device()
    out_dir = os.path.join(ROOT, "variants", name)
    os.makedirs(out_dir, exist_ok=True)
    srcp = src if os.sep in src else os.path.join(B.DEV_SRC, src)  # a path: an alternative copy of a device TU
    src = os.path.basename(srcp)
    obj = os.path.join(out_dir, src + ".o")
    subprocess.run([B.NVCC, *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler",
                    "-fPIC", "-I", B.INC, "-I", B.DEV_SRC, "-I", B.HOST_SRC, *defs, "-c", srcp, "-o", obj], check=True)
    objs = [o for o in glob.glob(os.path.join(B.OBJ, "*.o")) if os.path.basename(o) != src + ".o"] + [obj]
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o",
                    os.path.join(out_dir, "libpf_device.so"), "-lcudart", f"-L{B.LIB}", "-lpf_host", "-Xlinker",
                    "-rpath=$ORIGIN/../../paper_2602_05754_b200/lib", *B._nccl_flags()], check=True)
    os.remove(obj)
    print(os.path.join(out_dir, "libpf_device.so"))


if __name__ == "__main__":
    main()
