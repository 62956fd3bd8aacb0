"""Opcode statistics of one kernel's SASS (run here, no GPU needed).

    python tools/sass_stats.py <substring of the mangled kernel name> [--list] [--dump out.sass]

Reads `cuobjdump -sass` of the built library; prints registers / stack, the opcode histogram of the whole function and
of its hottest loop (the longest backward-branch span), and the spill instructions if any.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2011_03479_b200", "lib", "libgempe_b200.so")


def functions():
    text = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    out, name, body = {}, None, []
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                out[name] = body
            name, body = m.group(1), []
        elif name and re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", line):
            body.append(line)
    if name:
        out[name] = body
    return out


def opcode(line):
    m = re.search(r"/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if not m:
        return None, None
    parts = m.group(2).split()
    op = parts[1] if parts[0].startswith("@") else parts[0]
    return int(m.group(1), 16), op


if __name__ == "__main__":
    fns = functions()
    if "--list" in sys.argv:
        print("\n".join(sorted(fns)))
        sys.exit(0)
    key = sys.argv[1]
    names = [n for n in fns if key in n]
    assert len(names) == 1, names
    body = fns[names[0]]
    if "--dump" in sys.argv:
        open(sys.argv[sys.argv.index("--dump") + 1], "w").write("\n".join(body))
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", LIB], capture_output=True, text=True).stdout.splitlines()
    for i, line in enumerate(res):
        if names[0] in line:
            print(res[i + 1].strip())
    ops = [opcode(l) for l in body]
    ops = [(a, o) for a, o in ops if o]
    print(f"{len(ops)} instructions")
    # hottest loop guess: the longest span closed by a backward branch
    best = (0, 0)
    for a, o in ops:
        if o.startswith("BRA"):
            line = next(l for l in body if f"/*{a:04x}*/" in l)
            m = re.search(r"BRA\S*\s+(?:\S+,\s*)?`?\(?\.?L?_?x?_?(\w+)\)?|BRA\S*\s+.*?0x([0-9a-f]+)", line)
            tgt = re.search(r"0x([0-9a-f]+)\s*;", line)
            if tgt:
                t = int(tgt.group(1), 16)
                if t < a and a - t > best[1] - best[0]:
                    best = (t, a)
    for title, sel in (("whole function", ops), (f"longest loop [{best[0]:#x}, {best[1]:#x}]",
                                                  [(a, o) for a, o in ops if best[0] <= a <= best[1]])):
        hist = collections.Counter(o.split(".")[0] for _, o in sel)
        print(f"-- {title}: {len(sel)} instructions")
        print("   " + "  ".join(f"{k}={v}" for k, v in hist.most_common(28)))
    spills = [l.strip() for l in body if re.search(r"\b(STL|LDL)", l)]
    print(f"-- local-memory instructions: {len(spills)}")
    for l in spills[:12]:
        print("   " + re.sub(r"\s+/\*[0-9a-fx]+\*/$", "", l))
