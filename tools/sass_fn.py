"""Dev tool (CPU): SASS of the kernels whose mangled name contains a substring.
    python tools/sass_fn.py <object or .so> <substring> [> out.sass]"""
import subprocess
import sys

obj, sub = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
keep = False
for line in out.splitlines():
    if line.strip().startswith("Function :"):
        keep = sub in line
    if keep and not line.strip().startswith("/* 0x"):
        print(line)
