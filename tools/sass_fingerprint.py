"""Fingerprints of the tuned kernels' SASS (their speed hangs on ptxas's register
assignment): any source change that perturbs them shows up here before
it costs GPU time.  usage: python tools/sass_fingerprint.py [--check]  (tools/sass_fingerprints.txt)"""
import hashlib
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_1401_6124_b200" / "lib" / "libmhb.so"
REF = ROOT / "tools" / "sass_fingerprints.txt"
KERNELS = {
    "cfg1-3,5 iterative (K=64)": "_ZN3mhb11sign_kernelILi64ELb1ELb1EjLb0ELb0ELb0EEEvNS_8SignArgsEjjjj",
    "cfg4 iterative (K=64, skew)": "_ZN3mhb11sign_kernelILi64ELb1ELb1EjLb0ELb0ELb1EEEvNS_8SignArgsEjjjj",
    "cfg4 fused band keys": "_ZN3mhb11sign_kernelILi64ELb1ELb1EjLb1ELb0ELb1EEEvNS_8SignArgsEjjjj",
    "random float-quotient (K=16)": "_ZN3mhb11sign_kernelILi16ELb0ELb1EjLb0ELb1ELb0EEEvNS_8SignArgsEjjjj",
    "random Shoup (K=16)": "_ZN3mhb11sign_kernelILi16ELb0ELb1EjLb0ELb0ELb0EEEvNS_8SignArgsEjjjj",
}


def fingerprints():
    out = {}
    for label, fn in KERNELS.items():
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, str(LIB)], capture_output=True, text=True).stdout
        ins = re.findall(r"/\*[0-9a-f]{4,5}\*/\s+([^;]+);", sass)
        out[label] = hashlib.sha256("\n".join(ins).encode()).hexdigest()[:16] if ins else "missing"
    return out


if __name__ == "__main__":
    fp = fingerprints()
    if "--check" in sys.argv:
        ref = dict(l.split("\t") for l in REF.read_text().splitlines() if "\t" in l)
        bad = [k for k, v in fp.items() if ref.get(k) != v]
        for k in fp:
            print(("CHANGED " if k in bad else "same    ") + k)
        sys.exit(1 if bad else 0)
    REF.write_text("".join(f"{k}\t{v}\n" for k, v in fp.items()))
    print(REF.read_text())
