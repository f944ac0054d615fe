"""Static SASS statistics per kernel of an object/library: instruction count and opcode histogram.
Usage: python scripts/sass_stats.py <file.o|.so> [name-substring] [--ops N]"""
import collections
import re
import subprocess
import sys


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if m and cur:
            body.append(m.group(1))
    if cur:
        yield cur, body


def main():
    path = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ""
    nops = int(sys.argv[sys.argv.index("--ops") + 1]) if "--ops" in sys.argv else 0
    for name, body in functions(path):
        if sub not in name:
            continue
        ops = collections.Counter()
        for ins in body:
            toks = ins.split()
            op = toks[1] if toks[0].startswith("@") else toks[0]
            ops[op.split(".")[0]] += 1
        print(f"{len(body):6d} {name}")
        if nops:
            print("       " + "  ".join(f"{o}:{c}" for o, c in ops.most_common(nops)))


main()
