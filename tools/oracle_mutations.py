#!/usr/bin/env python
"""Mutation check of the oracle pins: each plausible mistake, applied to a copy
of oracle/piko_oracle.c, must make tests/test_oracle_pins.py fail."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "piko_oracle.c")
MUTATIONS = [
    ("top-left rule inverted", "return (Yb == Ya && Xb > Xa) || (Yb < Ya);",
     "return (Yb == Ya && Xb < Xa) || (Yb > Ya);"),
    ("z plane operands transposed", "float a = fmaf(dz1, dy2, -(dz2 * dy1)) * inv;",
     "float a = fmaf(dz2, dx1, -(dz1 * dx2)) * inv;"),
    ("perspective weight dropped", "float l0 = ((float)w0 * inv) * o->rw[0];",
     "float l0 = ((float)w0 * inv);"),
    ("y not flipped", "float sy = fmaf(-yn, hh, hh);", "float sy = fmaf(yn, hh, hh);"),
    ("rank ownership ignored", "if (b % nranks == rank) count[b] += 1;", "count[b] += 1;"),
    ("pixel rect floor/ceil swapped", "int64_t px1 = floor_div256((int64_t)maxX - HALF_SAMPLE);",
     "int64_t px1 = ceil_div256((int64_t)maxX - HALF_SAMPLE);"),
    ("tie-break reversed", "if (key < K[p]) K[p] = key;",
     "if ((key >> 32) < (K[p] >> 32) || ((key >> 32) == (K[p] >> 32) && (uint32_t)key > (uint32_t)K[p]) || K[p] == CLEAR_KEY) K[p] = key;"),
    ("depth range test dropped", "if (!(z >= 0.0f && z <= 1.0f)) continue;", ""),
    ("clamp dropped", "lam = (q > 0.0f) ? q : 0.0f;", "lam = q;"),
    ("guard band deleted", "if (!(fabsf(fx) <= GUARD_BAND && fabsf(fy) <= GUARD_BAND)) return 0;", ""),
    ("guard band widened to 2^24", "#define GUARD_BAND 4194304.0f", "#define GUARD_BAND 16777216.0f"),
    ("near epsilon zero", "#define W_EPS 1e-6f", "#define W_EPS 0.0f"),
    ("snap ties away from zero", "*X = (int32_t)rintf(fx);", "*X = (int32_t)roundf(fx);"),
    ("zero-area cull removed", "if (area2 == 0) return;", ""),
    ("depth range open at zero", "if (!(z >= 0.0f && z <= 1.0f)) continue;", "if (!(z > 0.0f && z <= 1.0f)) continue;"),
]
# Semantically equivalent under IEEE round-to-nearest (no input reaches it):
# the plane z = fma(a, dx, fma(b, dy, zw0)) is -0.0 only if zw0 is -0.0, and
# zw0 = fma(zn, 0.5, 0.5) is never -0.0 (an exact zero sum rounds to +0.0).
EQUIVALENT = [("-0 key mask dropped", "((uint64_t)(float_bits(z) & 0x7FFFFFFFu) << 32)",
               "((uint64_t)float_bits(z) << 32)")]
src = open(SRC).read()
ok = True
for name, old, new in MUTATIONS:
    assert old in src, name
    path = f"/tmp/oracle_mut_{os.getpid()}.c"
    lib = path[:-2] + ".so"
    open(path, "w").write(src.replace(old, new))
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99",
                           "-fPIC", "-shared", path, "-o", lib, "-lm"])
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-x",
                        "-p", "no:cacheprovider"], cwd=ROOT, env={**os.environ, "ORACLE_LIB": lib},
                       capture_output=True, text=True)
    caught = r.returncode != 0
    ok &= caught
    print(f"{'caught' if caught else 'MISSED':7s} {name}: {r.stdout.strip().splitlines()[-1]}")
for name, old, new in EQUIVALENT:
    assert old in src, name
    path = f"/tmp/oracle_mut_{os.getpid()}.c"
    lib = path[:-2] + ".so"
    open(path, "w").write(src.replace(old, new))
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99",
                           "-fPIC", "-shared", path, "-o", lib, "-lm"])
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q",
                        "-p", "no:cacheprovider"], cwd=ROOT, env={**os.environ, "ORACLE_LIB": lib},
                       capture_output=True, text=True)
    print(f"equiv.  {name} (unreachable under IEEE RN, see comment): {r.stdout.strip().splitlines()[-1]}")
sys.exit(0 if ok else 1)
