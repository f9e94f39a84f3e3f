"""Build an A/B variant of libflashmask.so with extra nvcc defines into ablibs/<name>.so
(for scripts/ab_libs.py; the product build is paper_2410_01359_b200/build.py):

    python scripts/build_variant.py NAME [-DMACRO=VALUE ...]"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2410_01359_b200 import build as b  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "ablibs")
    objdir = os.path.join(out, "build_" + name)
    os.makedirs(objdir, exist_ok=True)
    cc = b.nvcc()

    def one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [cc, *b.ARCH, *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(len(b.SOURCES)) as ex:
        objs = list(ex.map(one, b.SOURCES))
    lib = os.path.join(out, name + ".so")
    subprocess.run([cc, *b.ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fPIC"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
