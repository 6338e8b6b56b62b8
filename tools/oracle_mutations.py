"""Mutation run for the oracle pins: each entry applies one plausible mistake to oracle/fb_oracle.c, builds the
mutant into /tmp, runs the CPU pin suite (tests/test_oracle_pins.py) against it (ORACLE_LIB) and records
which pins fail.  A mutation that no pin catches is a hole in the pins.

    python tools/oracle_mutations.py [out.txt]
"""
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "fb_oracle.c")
sys.path.insert(0, ROOT)
from oracle.oracle import CFLAGS  # noqa: E402  (same flags as the real build)

# (name, passage, exact text, replacement, occurrence to replace (0-based) or None = all)
MUTATIONS = [
    ("upsample: no sub-cell offset", "P:51, D7",
     "Ff[2 * i] = clampi(2 * Fc[2 * j] + (r - 2 * rc), 0, h - 1);\n            Ff[2 * i + 1] = clampi(2 * Fc[2 * j + 1] + (c - 2 * cc), 0, w - 1);",
     "Ff[2 * i] = clampi(2 * Fc[2 * j], 0, h - 1);\n            Ff[2 * i + 1] = clampi(2 * Fc[2 * j + 1], 0, w - 1);", None),
    ("upsample: no x2", "P:51, D7",
     "clampi(2 * Fc[2 * j] + (r - 2 * rc), 0, h - 1)", "clampi(Fc[2 * j] + (r - 2 * rc), 0, h - 1)", None),
    ("upsample: odd edge reuses the wrong coarse cell", "P:51, D7",
     "int rc = (r >> 1) < hc - 1 ? (r >> 1) : hc - 1;", "int rc = (r >> 1) < hc - 1 ? (r >> 1) : hc - 2;", None),
    ("upsample: output clamped one short", "P:51, D7/D10",
     "clampi(2 * Fc[2 * j + 1] + (c - 2 * cc), 0, w - 1)", "clampi(2 * Fc[2 * j + 1] + (c - 2 * cc), 0, w - 2)", None),
    ("hand-off: coarse dims swapped", "P:51, D7",
     "orc_upsample(tmp, hc, wc, F, h, w);", "orc_upsample(tmp, wc, hc, F, h, w);", None),
    ("init: h and w swapped", "P:48, D8",
     "F[2 * i] = (int32_t)mulhi32(u[0], (uint32_t)h);", "F[2 * i] = (int32_t)mulhi32(u[0], (uint32_t)w);", None),
    ("init: level missing from the Philox counter", "D21",
     "orc_draw(cfg->seed, (uint32_t)i, 0, (uint32_t)k, 0, 0,", "orc_draw(cfg->seed, (uint32_t)i, 0, 0u, 0, 0,", None),
    ("propagation: sign flipped", "P:72, D11",
     "int sr = clampi(F[2 * j] - dx, 0, h - 1), sc = clampi(F[2 * j + 1] - dy, 0, w - 1);",
     "int sr = clampi(F[2 * j] + dx, 0, h - 1), sc = clampi(F[2 * j + 1] + dy, 0, w - 1);", None),
    ("select: <= instead of <", "P:56, D16", "if (e < E[i]) {", "if (e <= E[i]) {", None),
    ("patch distance: one tap column dropped", "P:66-68, D20",
     "for (int dc = -p; dc <= p; ++dc)\n            for (int ch = 0; ch < 3; ++ch) {",
     "for (int dc = -p; dc < p; ++dc)\n            for (int ch = 0; ch < 3; ++ch) {", None),
    ("patch distance: operands transposed in the target index", "P:66-68",
     "float delta = px(B, h, w, r + dr, c + dc, ch) - px(A, h, w, sr + dr, sc + dc, ch);",
     "float delta = px(B, h, w, r + dc, c + dr, ch) - px(A, h, w, sr + dr, sc + dc, ch);", None),
    ("loss: alpha on the style term", "P:116, Eq. 3", "return fmaf(L->alpha, dg, ds);", "return fmaf(L->alpha, ds, dg);", None),
    ("remap: divides by (2p+1)^2 (Alg. 2 literal) instead of the valid count", "P:96-101, D19",
     "out[3 * ((size_t)r * w + c) + ch] = acc[ch] / (float)n;",
     "out[3 * ((size_t)r * w + c) + ch] = acc[ch] / (float)((2 * p + 1) * (2 * p + 1));", None),
    ("T-bar: self term dropped", "Eq. 7, D27",
     "members[2 * nm] = st->tasks[t].tgt_id; members[2 * nm + 1] = -1; ++nm;", "", None),
    ("blending table: wrong BT scale", "Alg. 4, D25", "b[e] = (prev[e] + rt[cid][e] * scale) * 0.5f;",
     "b[e] = (prev[e] + rt[cid][e]) * 0.5f;", None),
    ("Eq. 9: weights swapped", "P:266, D28", "o[e] = fmaf(xl[e], wl, xr[e] * wr);", "o[e] = fmaf(xl[e], wr, xr[e] * wl);", None),
    ("random search: odd steps reuse the even step's words", "D21",
     "int ox = (int)mulhi32(u[2 * (s & 1)], (uint32_t)(2 * R + 1)) - R;", "int ox = (int)mulhi32(u[0], (uint32_t)(2 * R + 1)) - R;", None),
    ("blend tracking: link to the neighbouring source instead of target", "P:259, D44",
     "if (tasks[b].src_id == j) { if (z == 0)", "if (tasks[b].src_id == j + (z == 0 ? -1 : 1)) { if (z == 0)", None),
    ("blend tracking: readout from the requested index instead of the target's", "P:259, D44",
     "int t0 = first[cfg->tracking ? i : q];", "int t0 = first[q];", None),
]


def run(out_path):
    src = open(SRC).read()
    lines = [f"oracle mutation run ({time.strftime('%Y-%m-%d %H:%M')}), pins = tests/test_oracle_pins.py (CPU)", ""]
    holes = 0
    with tempfile.TemporaryDirectory() as td:
        for name, cite, old, new, occ in MUTATIONS:
            n = src.count(old)
            if n == 0:
                lines.append(f"[SKIP] {name}: pattern not found (oracle changed?)")
                holes += 1
                continue
            mut = src.replace(old, new)
            cfile, lib = os.path.join(td, "m.c"), os.path.join(td, f"m{len(lines)}.so")
            open(cfile, "w").write(mut)
            subprocess.check_call(["gcc", *CFLAGS, "-o", lib, cfile, "-lm"])
            env = dict(os.environ, ORACLE_LIB=lib)
            t0 = time.time()
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-p", "no:cacheprovider",
                                "--timeout", "300", "-x" if os.environ.get("MUT_FAST") else "-q"],
                               cwd=ROOT, env=env, capture_output=True, text=True)
            failed = sorted({ln.split(" ")[1].split("::")[1].split("[")[0] for ln in r.stdout.splitlines()
                             if ln.startswith("FAILED ") or ln.startswith("ERROR ")})
            caught = r.returncode != 0
            holes += 0 if caught else 1
            lines.append(f"[{'CAUGHT' if caught else 'MISSED'}] {name} ({cite}; {n} site{'s' if n > 1 else ''}), "
                         f"{time.time() - t0:.0f} s")
            lines.append("    failing pins: " + (", ".join(failed) if failed else "none"))
            print(lines[-2], flush=True)
    lines += ["", f"{len(MUTATIONS) - holes} of {len(MUTATIONS)} mutations caught"]
    open(out_path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return holes


if __name__ == "__main__":
    sys.exit(1 if run(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_oracle_mutations.txt") else 0)
