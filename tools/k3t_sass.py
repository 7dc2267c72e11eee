"""Flops per HT term of the tabulated-kbar kernel k3t, read from its SASS.

Finds each k3t instantiation in libeucalc.so (cuobjdump -sass), takes its
hottest loop (the backward branch whose body holds the most shared-memory
loads: the unrolled term loop), and counts the floating-point instructions of
one trip. Every term has exactly one IDP (the DP4A/DP2A table index), so
terms per trip = IDP count. FFMA/DFMA count 2 flops, FADD/FMUL/DADD/DMUL 1. Prints one JSON line per instantiation.

  python tools/k3t_sass.py [path/to/libeucalc.so]
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2405_02256_b200", "libeucalc.so")
FLOPS = {"FFMA": 2, "FADD": 1, "FMUL": 1, "DFMA": 2, "DADD": 1, "DMUL": 1}


def functions(sass):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


def instructions(body):
    out = []
    for line in body:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            out.append((int(m.group(1), 16), m.group(2).strip()))
    return out


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    for name, body in functions(sass):
        if "k3t" not in name:
            continue
        ins = instructions(body)
        addr = {a: i for i, (a, _) in enumerate(ins)}
        best = None
        for i, (a, txt) in enumerate(ins):
            m = re.search(r"\bBRA\b.*?(0x[0-9a-f]+)", txt)
            if not m:
                continue
            tgt = int(m.group(1), 16)
            if tgt >= a or tgt not in addr:
                continue
            loop = [t for _, t in ins[addr[tgt]:i + 1]]
            lds = sum(1 for t in loop if re.search(r"\bLDS", t))
            if best is None or lds > best[0]:
                best = (lds, loop)
        if not best:
            continue
        ops = {}
        for t in best[1]:
            op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
            ops[op] = ops.get(op, 0) + 1
        flops = sum(FLOPS.get(k, 0) * v for k, v in ops.items())
        terms = ops.get("IDP", 0) or 1
        print(json.dumps({"kernel": name, "loop_instructions": len(best[1]), "terms_per_trip": terms,
                          "flops_per_term": flops / terms,
                          "ops_per_trip": {k: v for k, v in sorted(ops.items()) if k in FLOPS or k.startswith(("LDS", "IDP", "I2F"))}}))


if __name__ == "__main__":
    main()
