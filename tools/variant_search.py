"""Search semantically equivalent spellings of the iterative main loop for a
register assignment with fewer register-bank conflicts (build container, no GPU).

usage: python tools/variant_search.py [out_dir] [-j jobs]

Every combination of the source transformations below is written as a copy of
csrc/sign.cu, compiled to a cubin, and its cfg2 (K=64, no skew) and cfg4 (skewed)
kernels' main loops are scored: instruction count and the number of extra distinct
registers per bank (index mod 2) among the non-reused sources of each instruction
(`bank_conflicts`).  On the committed loop that score separates the variants A/B'd so
far: 68 for the committed loop; 99 for the opaque-operand variant,
which ran 3.4% slower.  The best candidates then go to `tools/build_variant.sh` +
`tools/ab.sh` on the GPU.
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
KERNELS = (("cfg2", FN_CFG2),  # also cfg1 / cfg3 iterative
           ("cfg4", FN_CFG4),
           ("cfg5", "_ZN3mhb11sign_kernelILi64ELb1ELb0EjLb0ELb0ELb0EEEvNS_8SignArgsEjjj"),
           ("rfpq", "_ZN3mhb11sign_kernelILi16ELb0ELb1EjLb0ELb1ELb0EEEvNS_8SignArgsEjjj"),
           ("rshoup", "_ZN3mhb11sign_kernelILi16ELb0ELb1EjLb0ELb0ELb0EEEvNS_8SignArgsEjjj"))

WALK_MIN3 = ("            best[k] = __vimin3_u32(best[k], ha, hb);\n"
             "            best[k + 1] = __vimin3_u32(best[k + 1], ga, gb);\n")
LOOP_BODY = ("                qa = __ldg(base + min(o, last));  // smaller sets of the group clamp to their last id\n"
             "                qb = __ldg(base + min(o + 1, last));\n"
             "                maxid = __vimax3_u32(maxid, xa, xb);\n"
             "                round2<K, ITER, NARROW, false, FPQ>(best, ls, xa, xb, p, bpar);\n")
BOUNDS = "__global__ void __launch_bounds__(kBlock, 2) sign_kernel("


def opaque_one(s):
    """Kernel parameter `one` (= 1): an operand ptxas cannot constant-fold."""
    s = s.replace("sign_kernel(SignArgs A, uint32_t p, uint32_t bpar, uint32_t negp) {",
                  "sign_kernel(SignArgs A, uint32_t p, uint32_t bpar, uint32_t negp, uint32_t one) {")
    s = s.replace("using SignKernelFn = void (*)(SignArgs, uint32_t, uint32_t, uint32_t);",
                  "using SignKernelFn = void (*)(SignArgs, uint32_t, uint32_t, uint32_t, uint32_t);")
    s = s.replace("fn<<<(unsigned)blocks, kBlock, smem, st>>>(A, A.p, A.b, 0u - A.p);",
                  "fn<<<(unsigned)blocks, kBlock, smem, st>>>(A, A.p, A.b, 0u - A.p, 1u);")
    s = s.replace("    LaneState<K, ITER> ls;\n    ls.negp = negp;",
                  "    LaneState<K, ITER> ls;\n    ls.negp = negp;\n    ls.one = one;")
    s = s.replace("    uint32_t negp;  // 2^32 - p (kernel parameter; random family only)",
                  "    uint32_t negp;  // 2^32 - p (kernel parameter; random family only)\n    uint32_t one;")
    return s


ADDR_HELPER = """
__device__ __forceinline__ uint32_t ld_id(const uint32_t* base, uint32_t j, uint32_t four) {
    const uint32_t* a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(j), "r"(four), "l"(base));
    return __ldg(a);
}

// Per-thread hashing state"""

START_HELPER = """
template <int K, bool ITER>
__device__ __forceinline__ uint32_t start_hash_min3(const LaneState<K, ITER>& ls, uint32_t x) {
    const uint32_t q = __umulhi(ls.tAp, x);
    const uint32_t r = ls.tA * x + ls.tB + q * ls.negp;
    return __vimin3_u32(r, r * ls.one + ls.negp, r * ls.one + 2u * ls.negp);
}

template <int K, bool ITER, bool NARROW, bool FIRST, bool FPQ = false>
__device__ __forceinline__ void round2("""


def transform(src, min3_order, loads_swapped, maxid_after, features_swapped, maxnreg, addr=0, start=0):
    s = src
    assert WALK_MIN3 in s and LOOP_BODY in s and BOUNDS in s
    if addr or start:
        s = opaque_one(s)
    if addr:
        s = s.replace("\n// Per-thread hashing state", ADDR_HELPER, 1)
        s = s.replace("    const int F = A.F;\n    const int g = lane >> A.log2F;",
                      "    const uint32_t four = one << 2;\n    const int F = A.F;\n    const int g = lane >> A.log2F;")
    if start:
        s = s.replace("\ntemplate <int K, bool ITER, bool NARROW, bool FIRST, bool FPQ = false>\n"
                      "__device__ __forceinline__ void round2(", START_HELPER, 1)
        for x in ("xa", "xb"):
            s = s.replace(f"NARROW ? mul_add_mod_min3(ls.tA, ls.tAp, ls.tB, {x}, p)",
                          f"NARROW ? start_hash_min3(ls, {x})")
    if min3_order:
        s = s.replace(WALK_MIN3, "            best[k] = __vimin3_u32(ha, hb, best[k]);\n"
                                 "            best[k + 1] = __vimin3_u32(ga, gb, best[k + 1]);\n")
    if addr:
        la = "                qa = ld_id(base, min(o, last), four);\n"
        lb = "                qb = ld_id(base, min(o + 1, last), four);\n"
    else:
        la = "                qa = __ldg(base + min(o, last));  // smaller sets of the group clamp to their last id\n"
        lb = "                qb = __ldg(base + min(o + 1, last));\n"
    mx = "                maxid = __vimax3_u32(maxid, xa, xb);\n"
    rd = ("                round2<K, ITER, NARROW, false, FPQ>(best, ls, xb, xa, p, bpar);\n" if features_swapped
          else "                round2<K, ITER, NARROW, false, FPQ>(best, ls, xa, xb, p, bpar);\n")
    loads = lb + la if loads_swapped else la + lb
    body = loads + (rd + mx if maxid_after else mx + rd)
    s = s.replace(LOOP_BODY, body)
    if maxnreg:
        s = s.replace(BOUNDS, f"__global__ void __maxnreg__({maxnreg}) sign_kernel(")
    return s


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


ALU_OPS = ("VIADDMNMX", "VIMNMX3", "VIMNMX", "IADD3", "LEA", "ISETP", "LOP3", "SEL", "SHF", "IMNMX", "PLOP3")


def alu_count(ins):
    """Instructions that issue to the ALU pipe (B300_MICROARCH.md: IADD3/LOP3/SHF/... on alu)."""
    return sum(1 for t in ins if t.split()[0].lstrip("@!P0123456789").split(".")[0] in ALU_OPS
               or (t.startswith("@") and t.split()[1].split(".")[0] in ALU_OPS))


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
    combos = list(itertools.product([0, 1], [0, 1], [0, 1], [0, 1], [0, 120], [0, 1], [0, 1]))
    tasks = []
    for c in combos:
        name = "v_" + "".join(str(int(bool(x))) for x in c[:4]) + f"_{c[4]}_" + f"{c[5]}{c[6]}"
        tasks.append((name, transform(src, *c)))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda t: build_one(out_dir, *t), tasks))
    results.sort(key=lambda r: (r[1]["cfg2"][2], r[1]["cfg2"][1]))
    print("variant          " + "".join(f"{k:>18s}" for k, _ in KERNELS) + "   (inst, ALU, bank conflicts)")
    for name, r in results:
        print(f"{name:16s} " + "".join(f"{str(r[k]):>18s}" for k, _ in KERNELS))


if __name__ == "__main__":
    main()
