"""Per-function SASS statistics of a cubin/.so (instruction count, opcode mix).
Usage: python tools/sass_stats.py paper_2410_22205_b200/liblsr_b200.so [substring]"""
import collections
import re
import subprocess
import sys


def parse(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if m and cur:
            ins = m.group(1).strip()
            ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
            funcs[cur].append(ins.split()[0])
    return funcs


def main():
    funcs = parse(sys.argv[1])
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    for f, ins in funcs.items():
        if pat not in f:
            continue
        c = collections.Counter(i.split(".")[0] for i in ins)
        top = ", ".join(f"{k} {v}" for k, v in c.most_common(18))
        print(f"{len(ins):6d}  {f}\n        {top}")


if __name__ == "__main__":
    main()
