"""Static SASS instruction mix of kernels in an object / cubin / .so
(usage: python tools/sass_mix.py FILE [substring ...]).  Counts every
instruction of each matching function; FMA-pipe (IMAD*), ALU-pipe and
shared/global memory classes are summed for a quick pipe-balance check."""
import collections
import re
import subprocess
import sys

FMA = ("IMAD", "FFMA", "FMUL")
ALU = ("IADD3", "VIADDMNMX", "VIADD", "IMNMX", "VIMNMX", "LOP3", "SHF", "SEL", "ISETP", "LEA", "PRMT", "IABS", "MOV",
       "FMNMX", "FSEL", "PLOP3", "SGXT", "BMSK")


def main():
    path, subs = sys.argv[1], sys.argv[2:]
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if subs and not any(s in name for s in subs):
            continue
        ops = collections.Counter()
        for line in f.split("\n"):
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                ops[m.group(2)] += 1
        tot = sum(ops.values())
        fma = sum(n for o, n in ops.items() if o.startswith(FMA))
        alu = sum(n for o, n in ops.items() if o.split(".")[0] in ALU)
        lds = sum(n for o, n in ops.items() if o.startswith(("LDS", "STS")))
        gmem = sum(n for o, n in ops.items() if o.startswith(("LDG", "STG")))
        print(f"{name}\n  total {tot}  fma-pipe {fma}  alu-pipe {alu}  smem {lds}  gmem {gmem}")
        print("  " + ", ".join(f"{o}:{n}" for o, n in ops.most_common(18)))


if __name__ == "__main__":
    main()
