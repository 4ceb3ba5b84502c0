"""Build an A/B variant of libhd.so with a sed-style substitution in one source file.

    python tools/build_variant.py NAME FILE 'OLD' 'NEW' ['OLD' 'NEW' ...]  -> paper_2604_00546_b200/libhd_NAME.so
Use with HD_LIBHD=paper_2604_00546_b200/libhd_NAME.so python bench.py ...
"""
import glob
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_00546_b200", "csrc")


def main():
    name, fname = sys.argv[1:3]
    pairs = list(zip(sys.argv[3::2], sys.argv[4::2]))  # one or more OLD NEW substitutions
    tmp = tempfile.mkdtemp()
    dst = os.path.join(tmp, "pkg", "csrc")  # the sources include ../../include/hd.h
    shutil.copytree(CSRC, dst)
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    src = open(os.path.join(dst, fname)).read()
    for old, new in pairs:
        assert old in src, f"pattern not found in {fname}: {old}"
        src = src.replace(old, new)
    open(os.path.join(dst, fname), "w").write(src)
    objs = []
    procs = []
    for f in sorted(glob.glob(os.path.join(dst, "*.cu"))):
        o = f[:-3] + ".o"
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
               "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-O3",
               "-c", f, "-o", o]
        procs.append(subprocess.Popen(cmd))
        objs.append(o)
    for p in procs:
        assert p.wait() == 0
    out = os.path.join(ROOT, "paper_2604_00546_b200", f"libhd_{name}.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs,
                           "-lcudart"])
    shutil.rmtree(tmp)
    print(out)


if __name__ == "__main__":
    main()
