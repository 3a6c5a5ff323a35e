"""Print the SASS of the functions in a .so whose mangled name matches a regex.
Usage: python scripts/sass_fn.py lib.so REGEX"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2])
cur = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        if pat.search(cur):
            print(line)
        continue
    if cur and pat.search(cur):
        print(line)
