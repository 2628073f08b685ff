"""Dev helper: build a variant of libqapsa.so from a patched copy of csrc/ (the in-tree sources are
untouched): python tools/variant.py NAME PATCH.py -> variants/libqapsa_NAME.so, where PATCH.py
edits files under the copy (its root in the VROOT variable) by exact string replacement."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1208_2675_b200 import _build  # noqa: E402

name, patch = sys.argv[1], sys.argv[2]
vroot = f"/tmp/qapsa_var_{name}"
shutil.rmtree(vroot, ignore_errors=True)
shutil.copytree(os.path.join(ROOT, "paper_1208_2675_b200", "csrc"), os.path.join(vroot, "pkg", "csrc"))
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(vroot, "include"))
env = {"VROOT": vroot}
exec(open(patch).read(), env)
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", f"libqapsa_{name}.so")
cmd = [_build.nvcc(), *_build.NVCC_FLAGS, "-I", os.path.join(vroot, "include"), "-o", out,
       os.path.join(vroot, "pkg", "csrc", "qapsa.cu")]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stderr[-4000:])
print(out)
