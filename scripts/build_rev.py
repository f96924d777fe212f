"""Build the kernels of a git revision as an experiment variant (A/B timing on one box):
python scripts/build_rev.py REV NAME [DEF=V ...] -> paper_2101_11408_b200/libfpparse_NAME.so"""
import os, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_11408_b200 import build

rev, name = sys.argv[1], sys.argv[2]
build.build()  # generated tables in the tree are current
with tempfile.TemporaryDirectory() as d:
    arc = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_2101_11408_b200/csrc", "include"], check=True,
                         capture_output=True).stdout
    subprocess.run(["tar", "-x", "-C", d], input=arc, check=True)
    src = os.path.join(d, "paper_2101_11408_b200", "csrc")
    # generated (untracked) headers come from the current tree
    for f in os.listdir(build.CSRC):
        if not os.path.exists(os.path.join(src, f)):
            os.symlink(os.path.join(build.CSRC, f), os.path.join(src, f))
    out = os.path.join(build.HERE, "libfpparse_%s.so" % name)
    cmd = [build.NVCC] + build.ARCH + build.FLAGS + ["-D%s" % x for x in sys.argv[3:]] + [
        "-o", out, os.path.join(src, "fpparse.cu")]
    subprocess.check_call(cmd)
    print(out)
