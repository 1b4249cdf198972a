"""Opcode histogram of one kernel's SASS (cuobjdump -sass), optionally of
the instructions between two labels.  Diagnostic only.
    python tools/sass_hist.py <obj> <kernel-substring>"""
import collections
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = collections.Counter()
    for line in f.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            ops[m.group(2)] += 1
    print(name[:150], sum(ops.values()))
    print(" ".join(f"{k}:{v}" for k, v in ops.most_common(30)))
