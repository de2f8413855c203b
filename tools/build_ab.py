"""Build libils.so from a git revision into paper_2203_15340_b200/lib_<tag>/ for A/B timing with
ILS_LIB_PATH (development aid). usage: python tools/build_ab.py <rev> <tag>"""
import importlib.util
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rev, tag = sys.argv[1], sys.argv[2]
    tmp = tempfile.mkdtemp()
    arc = subprocess.run(["git", "archive", rev, "paper_2203_15340_b200/csrc", "include"], cwd=ROOT,
                         capture_output=True, check=True).stdout
    subprocess.run(["tar", "-x", "-C", tmp], input=arc, check=True)
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2203_15340_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.SRC = os.path.join(tmp, "paper_2203_15340_b200", "csrc")
    b.LIB_DIR = os.path.join(ROOT, "paper_2203_15340_b200", f"lib_{tag}")
    b.LIB = os.path.join(b.LIB_DIR, "libils.so")
    b.FLAGS = b.FLAGS[:-1] + [os.path.join(tmp, "include")]
    print(b.build(force=True))


if __name__ == "__main__":
    main()
