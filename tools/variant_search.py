"""Search the per-kernel loop spellings of csrc/sign.cu (`Spelling`) for register
assignments with fewer register-bank conflicts (build container, no GPU).

usage: python tools/variant_search.py [out_dir] [-j jobs]

The spellings are semantically identical; they only steer ptxas:
start-hash subtractions on the FMA pipe, id max after the round, features passed as
(b, a), IMAD.WIDE id addresses, and `__maxnreg__`.  Each combination is applied to
every kernel (the `Spelling` body is replaced), compiled to a cubin, and each kernel's
main loop is scored: instructions, ALU-pipe instructions, and bank conflicts — the
extra distinct registers with the same index mod 2 among an instruction's sources not
served by the reuse cache.  Kernels are separate instantiations, so the best row per
column can be combined per kernel class in `Spelling`.  The score is a filter: time
the candidates with tools/build_variant.sh + tools/ab.sh before committing one.

The first row is the committed source.
"""
import itertools
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1401_6124_b200", "csrc")
FN_CFG2 = "_ZN3mhb11sign_kernelILi64ELb1ELb1EjLb0ELb0ELb0EEEvNS_8SignArgsEjjj"
FN_CFG4 = "_ZN3mhb11sign_kernelILi64ELb1ELb1EjLb0ELb0ELb1EEEvNS_8SignArgsEjjj"
KERNELS = (("iter64", FN_CFG2),  # cfg1/2/3/5 iterative
           ("skew", FN_CFG4),  # cfg4
           ("rfpq", "_ZN3mhb11sign_kernelILi16ELb0ELb1EjLb0ELb1ELb0EEEvNS_8SignArgsEjjj"),  # cfg1/3 random
           ("rshoup", "_ZN3mhb11sign_kernelILi16ELb0ELb1EjLb0ELb0ELb0EEEvNS_8SignArgsEjjj"))  # cfg2 random
ALU_OPS = ("VIADDMNMX", "VIMNMX3", "VIMNMX", "IADD3", "LEA", "ISETP", "LOP3", "SEL", "SHF", "IMNMX", "PLOP3")


def spelling_body(start, maxid_after, swap, addr, maxnreg):
    return (f"    static constexpr bool kIter64 = ITER && NARROW && K == 64 && !BANDS;\n"
            f"    static constexpr bool start_fma = ITER && NARROW && {str(bool(start)).lower()};\n"
            f"    static constexpr bool maxid_after = {str(bool(maxid_after)).lower()};\n"
            f"    static constexpr bool swap_features = {str(bool(swap)).lower()};\n"
            f"    static constexpr bool addr_fma = {str(bool(addr)).lower()};\n"
            f"    static constexpr int maxnreg = {maxnreg};")


def transform(src, *flags):
    m = re.search(r"struct Spelling \{\n(.*?)\n\};", src, re.S)
    assert m, "Spelling struct not found"
    return src[:m.start(1)] + spelling_body(*flags) + src[m.end(1):]


def loop_instructions(sass, fn):
    i = sass.index("Function : " + fn)
    j = sass.find("Function : ", i + 10)
    body = sass[i:j if j > 0 else None]
    ins = [(int(m.group(1), 16), m.group(2).strip())
           for m in re.finditer(r"/\*([0-9a-f]{4,5})\*/\s+([^;]+);", body)]
    loops = []
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            lo = int(m.group(1), 16)
            sub = [x for b, x in ins if lo <= b <= a]
            loops.append((sum("VIADDMNMX" in x for x in sub) / len(sub), lo, a))
    loops.sort(reverse=True)
    _, lo, hi = loops[0]
    return [t for a, t in ins if lo <= a <= hi]


def bank_conflicts(ins, n_banks=2):
    total = 0
    for t in ins:
        parts = t.split(None, 1)
        if len(parts) < 2:
            continue
        by_bank = {}
        for o in [o.strip() for o in parts[1].split(",")][1:]:
            m = re.fullmatch(r"-?\|?R(\d+)(\.reuse)?\|?(\.\w+)*", o)
            if m and not m.group(2):
                by_bank.setdefault(int(m.group(1)) % n_banks, set()).add(int(m.group(1)))
        total += sum(len(v) - 1 for v in by_bank.values() if len(v) > 1)
    return total


def alu_count(ins):
    """Instructions that issue to the ALU pipe (B300_MICROARCH.md: IADD3/LOP3/SHF/... on alu)."""
    n = 0
    for t in ins:
        words = t.split()
        op = words[1] if words[0].startswith("@") else words[0]
        n += op.split(".")[0] in ALU_OPS
    return n


def build_one(out_dir, name, text):
    d = os.path.join(out_dir, name)
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, "sign.cu")
    cubin = os.path.join(d, "sign.cubin")
    fresh = os.path.exists(cubin) and os.path.exists(path) and open(path).read() == text
    if not fresh:  # (re)compile only what changed
        with open(path, "w") as f:
            f.write(text)
        subprocess.run(["nvcc", "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                        "--expt-relaxed-constexpr", f"-I{ROOT}/include", f"-I{SRC}", "-cubin", "-o", cubin, path],
                       check=True, capture_output=True)
    sass = subprocess.run(["cuobjdump", "-sass", cubin], check=True, capture_output=True, text=True).stdout
    res = {}
    for key, fn in KERNELS:
        ins = loop_instructions(sass, fn)
        res[key] = (len(ins), alu_count(ins), bank_conflicts(ins))
    return name, res


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "/tmp/variant_search"
    jobs = int(sys.argv[sys.argv.index("-j") + 1]) if "-j" in sys.argv else os.cpu_count()
    src = open(os.path.join(SRC, "sign.cu")).read()
    tasks = [("committed", src)]
    for c in itertools.product([0, 1], [0, 1], [0, 1], [0, 1], [128, 120]):
        tasks.append(("s" + "".join(map(str, c[:4])) + f"_{c[4]}", transform(src, *c)))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda t: build_one(out_dir, *t), tasks))
    print("spelling: start_fma maxid_after swap_features addr_fma _maxnreg; (instructions, ALU, bank conflicts)")
    print(f"{'variant':12s}" + "".join(f"{k:>18s}" for k, _ in KERNELS))
    for name, r in results:
        print(f"{name:12s}" + "".join(f"{str(r[k]):>18s}" for k, _ in KERNELS))


if __name__ == "__main__":
    main()
