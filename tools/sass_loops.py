"""Static schedule of a kernel's SASS loops: for every backward branch, the loop
body's instruction count, FP64 count and the sum of the encoded stall counts
(the minimum cycles one warp needs per iteration when nothing else stalls it).

    cuobjdump -sass -fun <mangled> lib.so > k.sass; python tools/sass_loops.py k.sass [--dump LO HI]

Control word (sm_70+ 128-bit encoding, high 64-bit word): stall = bits 41-44,
yield 45, write barrier 46-48, read barrier 49-51, wait mask 52-57.
"""
import re
import sys

FP64 = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")


def parse(path):
    ins = []
    lines = open(path).read().splitlines()
    i = 0
    pat = re.compile(r"^\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* 0x([0-9a-f]{16}) \*/")
    pat2 = re.compile(r"^\s*/\* 0x([0-9a-f]{16}) \*/")
    while i < len(lines):
        m = pat.match(lines[i])
        if m and i + 1 < len(lines):
            m2 = pat2.match(lines[i + 1])
            if m2:
                hi = int(m2.group(1), 16)
                ctrl = hi >> 41
                ins.append({"addr": int(m.group(1), 16), "text": m.group(2).strip(),
                            "stall": ctrl & 15, "yield": (ctrl >> 4) & 1, "wr": (ctrl >> 5) & 7,
                            "rd": (ctrl >> 8) & 7, "wait": (ctrl >> 11) & 63})
                i += 2
                continue
        i += 1
    return ins


def opcode(t):
    t = re.sub(r"^@!?U?P\d+\s+", "", t)
    return t.split()[0].split(".")[0]


def main():
    ins = parse(sys.argv[1])
    by_addr = {x["addr"]: k for k, x in enumerate(ins)}
    print(f"{len(ins)} instructions")
    if "--dump" in sys.argv:
        j = sys.argv.index("--dump")
        lo, hi = int(sys.argv[j + 1], 16), int(sys.argv[j + 2], 16)
        for x in ins:
            if lo <= x["addr"] <= hi:
                print(f"{x['addr']:05x} s{x['stall']:2d} {'Y' if x['yield'] else ' '} w{x['wr']} r{x['rd']} m{x['wait']:02x}  {x['text']}")
        return
    for k, x in enumerate(ins):
        m = re.search(r"\bBRA\S*\s+(?:[!U]*P\d+,\s*)?`\(\.L_x_\d+\)", x["text"])
        if not m:
            continue
    # branch targets are printed as labels; cuobjdump prints addresses with -sass? fall back on 0x addresses
    for k, x in enumerate(ins):
        m = re.search(r"BRA\S*.*?0x([0-9a-f]+)", x["text"])
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt <= x["addr"] and tgt in by_addr:
            body = ins[by_addr[tgt]:k + 1]
            n = len(body)
            f = sum(opcode(b["text"]) in FP64 for b in body)
            st = sum(max(b["stall"], 1) for b in body)
            ops = {}
            for b in body:
                ops[opcode(b["text"])] = ops.get(opcode(b["text"]), 0) + 1
            top = sorted(ops.items(), key=lambda kv: -kv[1])[:8]
            print(f"loop {tgt:05x}-{x['addr']:05x}: {n} instr, {f} fp64, stall sum {st}, "
                  f"{st / n:.2f} cyc/instr; {top}")


if __name__ == "__main__":
    main()
