#!/usr/bin/env python3
"""Static SASS opcode histogram of one kernel in a built object:
tools/sass_hist.py <object> <mangled-name-substring> [top]"""
import collections
import re
import subprocess
import sys


def kernels(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    cur, body = None, collections.defaultdict(list)
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?)\s*;", line)
        if m and cur:
            body[cur].append(m.group(1))
    return body


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    for name, ins in kernels(obj).items():
        if pat not in name:
            continue
        h = collections.Counter()
        for i in ins:
            i = re.sub(r"^@!?U?P\d+\s+", "", i)
            h[i.split()[0]] += 1
        print(f"{name}: {len(ins)} instructions")
        print("  " + ", ".join(f"{k} {v}" for k, v in h.most_common(top)))


if __name__ == "__main__":
    main()
