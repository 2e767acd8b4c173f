"""Build libsq.so from another git revision (or a directory) for A/B timing.

python tools/build_variant.py <rev> <name>      -> paper_2312_03788_b200/_lib/variants/libsq_<name>.so
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_03788_b200 import build as B  # noqa: E402


def main():
    rev, name = sys.argv[1], sys.argv[2]
    out_dir = os.path.join(ROOT, "paper_2312_03788_b200", "_lib", "variants")
    os.makedirs(out_dir, exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        for path in ("paper_2312_03788_b200/csrc", "include"):
            os.makedirs(os.path.join(td, path), exist_ok=True)
            files = subprocess.run(["git", "ls-tree", "--name-only", f"{rev}:{path}"], cwd=ROOT,
                                   capture_output=True, text=True, check=True).stdout.split()
            for f in files:
                data = subprocess.run(["git", "show", f"{rev}:{path}/{f}"], cwd=ROOT, capture_output=True,
                                      check=True).stdout
                with open(os.path.join(td, path, f), "wb") as fh:
                    fh.write(data)
        objs = []
        srcs = sorted(os.listdir(os.path.join(td, "paper_2312_03788_b200/csrc")))
        for f in srcs:
            if not f.endswith(".cu"):
                continue
            o = os.path.join(td, f[:-3] + ".o")
            flags = [x.replace(os.path.join(ROOT, "include"), os.path.join(td, "include")) for x in B.CFLAGS]
            subprocess.run([B.nvcc(), *flags, "-c", os.path.join(td, "paper_2312_03788_b200/csrc", f), "-o", o],
                           check=True)
            objs.append(o)
        lib = os.path.join(out_dir, f"libsq_{name}.so")
        subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-ldl", "-lrt",
                        "-lpthread"], check=True)
        print(lib)


if __name__ == "__main__":
    main()
