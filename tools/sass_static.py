"""Static SASS op mix of one kernel in an object/.so (no GPU needed).

    python tools/sass_static.py <file.o|.so> <mangled-name-substring> [top]
"""
import collections
import re
import subprocess
import sys


def main(path, pat, top=30):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if pat not in name:
            continue
        ops = collections.Counter()
        for line in f.split("\n"):
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
            if m:
                ops[m.group(2)] += 1
        print(name, sum(ops.values()))
        for k, v in ops.most_common(int(top)):
            print(f"  {k:12s} {v}")


if __name__ == "__main__":
    main(*sys.argv[1:])
