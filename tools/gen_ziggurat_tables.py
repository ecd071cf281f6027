"""Generate csrc/bwm_ziggurat_tables.h: the constants of numpy's standard-normal ziggurat.

The reference's critical_value draws its null series with
``np.random.Generator(np.random.Philox(key=seed, counter=r << 128)).standard_normal(N)``
(reference mosum.py:195-198).  numpy (a third-party dependency of the reference, pinned here at
the image's numpy 2.3) implements that as Philox4x64-10 (Random123) feeding the 256-layer
Marsaglia-Tsang ziggurat of numpy/random/src/distributions/distributions.c
(random_standard_normal).  The ziggurat's three 256-entry tables (ki: uint64 acceptance
thresholds, wi: layer widths, fi: layer heights) are data, not code; this script reads them
from the .rodata of numpy's own static library (numpy/random/lib/libnpyrandom.a, shipped for
Cython users), restates the published algorithm in Python, checks it reproduces numpy's
draws bit for bit, and writes the header.  Run once; the header is committed.

    python tools/gen_ziggurat_tables.py
"""
import os
import struct
import subprocess
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parents[1] / "paper_1807_01751_b200" / "csrc" / "bwm_ziggurat_tables.h"
M64 = (1 << 64) - 1
PHILOX_M0, PHILOX_M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
PHILOX_W0, PHILOX_W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
NOR_R = 3.6541528853610087963519472518
NOR_INV_R = 0.27366123732975827203338247596


def extract_tables():
    lib = Path(np.__file__).parent / "random" / "lib" / "libnpyrandom.a"
    with tempfile.TemporaryDirectory() as d:
        members = subprocess.run(["ar", "t", str(lib)], capture_output=True, text=True, check=True).stdout.split()
        member = next(m for m in members if "distributions.c" in m and "logfactorial" not in m)
        subprocess.run(["ar", "x", str(lib), member], cwd=d, check=True)
        obj = os.path.join(d, member)
        syms = {}
        for line in subprocess.run(["nm", obj], capture_output=True, text=True, check=True).stdout.splitlines():
            parts = line.split()
            if len(parts) == 3 and parts[2] in ("ki_double", "wi_double", "fi_double"):
                syms[parts[2]] = int(parts[0], 16)
        rod = os.path.join(d, "rodata.bin")
        subprocess.run(["objcopy", "-O", "binary", "--only-section=.rodata", obj, rod], check=True)
        data = Path(rod).read_bytes()
    ki = list(struct.unpack("<256Q", data[syms["ki_double"]: syms["ki_double"] + 2048]))
    wi = list(struct.unpack("<256d", data[syms["wi_double"]: syms["wi_double"] + 2048]))
    fi = list(struct.unpack("<256d", data[syms["fi_double"]: syms["fi_double"] + 2048]))
    return ki, wi, fi


def philox4x64_10(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for rnd in range(10):
        if rnd:
            k0, k1 = (k0 + PHILOX_W0) & M64, (k1 + PHILOX_W1) & M64
        p0, p1 = PHILOX_M0 * c[0], PHILOX_M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & M64, (p0 >> 64) ^ c[3] ^ k1, p0 & M64]
    return c


class Stream:
    """Philox(key=seed, counter=rep << 128) as numpy's bit generator consumes it."""

    def __init__(self, seed, rep):
        self.key = (seed & M64, (seed >> 64) & M64)
        c = rep << 128
        self.ctr = [(c >> (64 * i)) & M64 for i in range(4)]
        self.buf, self.pos = [0] * 4, 4

    def next64(self):
        if self.pos == 4:
            for i in range(4):                         # increment with carry, then encrypt
                self.ctr[i] = (self.ctr[i] + 1) & M64
                if self.ctr[i]:
                    break
            self.buf, self.pos = philox4x64_10(self.ctr, self.key), 0
        v = self.buf[self.pos]
        self.pos += 1
        return v

    def next_double(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def standard_normal(s, ki, wi, fi):
    while True:
        r = s.next64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            return x
        if idx == 0:
            while True:
                xx = -NOR_INV_R * np.log1p(-s.next_double())
                yy = -np.log1p(-s.next_double())
                if yy + yy > xx * xx:
                    return -(NOR_R + xx) if (rabs >> 8) & 1 else NOR_R + xx
        elif (fi[idx - 1] - fi[idx]) * s.next_double() + fi[idx] < np.exp(-0.5 * x * x):
            return x


def verify(ki, wi, fi):
    for seed, reps, n in ((7, 40, 300), (1, 12, 1000), (2**64 - 5, 5, 200)):
        for rep in range(reps):
            ref = np.random.Generator(np.random.Philox(key=seed, counter=rep << 128)).standard_normal(n)
            s = Stream(seed, rep)
            ours = np.array([standard_normal(s, ki, wi, fi) for _ in range(n)])
            assert np.array_equal(ours.view(np.uint64), ref.view(np.uint64)), (seed, rep)


def main():
    ki, wi, fi = extract_tables()
    verify(ki, wi, fi)
    lines = [
        "// bwm_ziggurat_tables.h — GENERATED by tools/gen_ziggurat_tables.py; do not edit.",
        f"// numpy {np.__version__} standard-normal ziggurat constants (random_standard_normal,",
        "// numpy/random/src/distributions/distributions.c), read from numpy's libnpyrandom.a and",
        "// checked there: the restated Philox4x64-10 + ziggurat reproduces numpy's draws bit for bit.",
        "#pragma once",
        "#include <stdint.h>",
        "namespace bwm {",
        "__constant__ uint64_t kZigKi[256] = {" + ", ".join(f"0x{v:016x}ull" for v in ki) + "};",
        "__constant__ double kZigWi[256] = {" + ", ".join(float.hex(v) for v in wi) + "};",
        "__constant__ double kZigFi[256] = {" + ", ".join(float.hex(v) for v in fi) + "};",
        "}  // namespace bwm",
        "",
    ]
    OUT.write_text("\n".join(lines))
    print(f"wrote {OUT} (verified against numpy {np.__version__})")


if __name__ == "__main__":
    main()
