"""Builds an A/B variant of libcorr.so: copies csrc/ to a temp dir, applies literal
replacements (pairs of strings), and links tools/ab/<name>.so.  Development tool."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_03308_b200 import build as B  # noqa: E402


def main(name, *subs):
    tmp = tempfile.mkdtemp()
    src = os.path.join(tmp, "csrc")
    shutil.copytree(B.CSRC, src)
    pairs = list(zip(subs[0::2], subs[1::2]))
    for fn in os.listdir(src):
        p = os.path.join(src, fn)
        s = open(p).read()
        for a, b in pairs:
            s = s.replace(a, b)
        open(p, "w").write(s)
    objs = []
    for fn in sorted(os.listdir(src)):
        if fn.endswith(".cu"):
            o = os.path.join(tmp, fn + ".o")
            flags = [f.replace(B.CSRC, src) for f in B.FLAGS]
            subprocess.check_call([B.NVCC, *B.ARCH, *flags, "-c", os.path.join(src, fn), "-o", o])
            objs.append(o)
    out = os.path.join(ROOT, "tools", "ab", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    print(out)


if __name__ == "__main__":
    main(*sys.argv[1:])
