"""Register/spill summary of the wave kernels from a verbose nvcc build log (development aid)."""
import re, sys
cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        n = re.sub(r"_ZN4sorb11wave_kernelI([df])Li(\d)ELi1[24]ELi(\d)ELb(\d)E(Li(\d)E)?E.*", r"wave<\1,T=\2,ck=\3,split=\4>", cur)
        if "wave" in n:
            print(f"{n:28s} regs {m.group(1):>4s}  spill st/ld {spill}")
        cur = None
