"""Mutation check of the oracle pins (CPU only).

Each mutant is a plausible mistake in oracle/*.c (a dropped term, a wrong sign
or index, a swapped operand, a non-inclusive comparison, a missing wrap...).
The mutant library is built from a patched copy and the CPU pin suites run
against it (ORACLE_MUTANT_LIB); every mutant must make at least one pin fail.

    python tools/mutate_oracle.py > profiles/r01_oracle_mutation.md
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_multi.py", "tests/test_oracle_list.py",
        "tests/test_instances_cpu.py", "tests/test_oracle_variants.py", "tests/test_oracle_flags.py",
        "tests/test_oracle_slab_r02.py"]

MUTANTS = [
    # (file, original, mutated, description)
    ("oracle.c", "o[0] = a[1] * b[2] - a[2] * b[1];", "o[0] = a[1] * b[2] + a[2] * b[1];",
     "cross product: wrong sign in x"),
    ("oracle.c", "o[1] = a[2] * b[0] - a[0] * b[2];", "o[1] = a[2] * b[1] - a[0] * b[2];",
     "cross product: wrong index in y"),
    ("oracle.c", "return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];",
     "return (a[0] * b[0] + a[1] * b[1]);", "dot product: dropped z term"),
    ("oracle.c", "cross3(d, e2, p);", "cross3(e2, d, p);", "MT: transposed cross operands (p)"),
    ("oracle.c", "*u = dot3(s, p) * inv;\n  cross3(s, e1, q);\n  *v = dot3(d, q) * inv;",
     "*v = dot3(s, p) * inv;\n  cross3(s, e1, q);\n  *u = dot3(d, q) * inv;", "MT: u and v swapped"),
    ("oracle.c", "(*u + *v <= 1.0f)", "(*u + *v < 1.0f)", "MT: edge test not inclusive"),
    ("oracle.c", "(*t >= tmin) && (*t <= tmax_cur)", "(*t > tmin) && (*t <= tmax_cur)",
     "MT: tmin not inclusive"),
    ("oracle.c", "if (!(fabsf(det) >= 1e-12f)) return 0;", "if (!(det >= 1e-12f)) return 0;",
     "MT: back faces culled"),
    ("oracle.c", "float w = (1.0f - u) - v;\n  out[0]", "float w = (1.0f - u);\n  out[0]",
     "lerp: dropped -v in the first weight"),
    ("oracle.c", "out[1] = (w * a[1] + u * b[1]) + v * c[1];", "out[1] = (w * a[1] + v * b[1]) + u * c[1];",
     "lerp: barycentrics swapped in t"),
    ("oracle.c", "return ((i % m) + m) % m;\n}\nfloat oracle_tex_alpha",
     "return i < 0 ? 0 : (i >= m ? m - 1 : i);\n}\nfloat oracle_tex_alpha", "tex2D: clamp instead of wrap"),
    ("oracle.c", "uint8_t a8 = rgba[((size_t)j * w + (size_t)i) * 4 + 3];",
     "uint8_t a8 = rgba[((size_t)i * h + (size_t)j) * 4 + 3];", "tex2D: transposed texel address"),
    ("oracle.c", "uint8_t a8 = rgba[((size_t)j * w + (size_t)i) * 4 + 3];",
     "uint8_t a8 = rgba[((size_t)j * w + (size_t)i) * 4 + 0];", "tex2D: red channel instead of alpha"),
    ("oracle.c", "return a >= thr;\n  }\n  if (isect == OR_ALPHA_PROC)", "return a > thr;\n  }\n  if (isect == OR_ALPHA_PROC)",
     "alpha threshold not inclusive"),
    ("oracle.c", "return ((cu + cv) % 2) == 0;", "return ((cu + cv) % 2) == 1;", "checker parity inverted"),
    ("oracle.c", "int cv = (int)floorf(v * fm);", "int cv = (int)floorf(u * fm);", "checker uses u twice"),
    ("oracle.c", "if (!have || t < best.t) {", "if (!have || t > best.t) {", "closest: keeps the farthest"),
    ("oracle.c", "    if (!filter(s, i, jb->isect, u, v, jb->thr, jb->M)) continue;\n    /* accepted */",
     "    /* accepted */", "filter ignored in the brute force"),
    ("oracle.c", "if (x->t < y->t) return -1;", "if (x->t > y->t) return -1;", "multi-hit sorted descending"),
    ("walker.c", "float tn = fmaxf(fmaxf(fminf(t0x, t1x), fminf(t0y, t1y)), fmaxf(fminf(t0z, t1z), tmin));",
     "float tn = fmaxf(fminf(t0x, t1x), fminf(t0y, t1y));", "slab: z slab and tmin dropped from tnear"),
    ("walker.c", "if (tn1 < tn0) { nearr = nd->ref[1]; farr = nd->ref[0]; ftn = tn0; }",
     "if (tn1 > tn0) { nearr = nd->ref[1]; farr = nd->ref[0]; ftn = tn0; }", "walker: far child first"),
    ("walker.c", "      c.boxes += 2;", "      c.boxes += 1;", "walker: one box count per inner node"),
    ("walker.c", "      if (st_tn[sp] > cull_bound(o, inv, best_t)) continue;", "", "walker: popped entries never culled"),
    ("walker.c", "  c.boxes++;\n  if (!slab(b->root_lo", "  if (!slab(b->root_lo", "walker: root test not counted"),
    ("walker.c", "        if (jb->isect == OR_ALPHA_TEX) c.alpha++;", "", "walker: alpha lookups not counted"),
    ("walker.c", "ax[a][c] = lo[a];\n    ax[a][2 + c] = hi[a];", "ax[a][2 + c] = lo[a];\n    ax[a][c] = hi[a];",
     "oracle BVH: lo/hi planes swapped in the node"),
    ("walker.c", "out[i] = ((r[0] * o[0] + r[1] * o[1]) + r[2] * o[2]) + r[3];",
     "out[i] = ((r[0] * o[0] + r[1] * o[1]) + r[2] * o[2]);", "instance map: translation dropped"),
    ("walker.c", "out[4 + i] = (r[0] * d[0] + r[1] * d[1]) + r[2] * d[2];",
     "out[4 + i] = (m[i] * d[0] + m[4 + i] * d[1]) + m[8 + i] * d[2];",
     "instance map: direction by the transposed matrix"),
    ("walker.c", "  S->c.boxes++;\n  if (!slab(b->root_lo", "  if (!slab(b->root_lo",
     "instances: bottom root test not counted"),
    ("walker.c", "if ((S->have && !had) || S->best_t < bt) *which = in->index;",
     "if ((S->have && !had) || S->best_t < bt) *which = k;",
     "instances: leaf position reported instead of the caller's index"),
    ("walker.c", "  return stop;\n}\n\nstatic void walk_instances_one", "  return 0;\n}\n\nstatic void walk_instances_one",
     "instances: any-hit keeps walking after a hit"),
    ("walker.c", "    if (fmaxf(fmaxf(fabsf(o[0]), fabsf(o[1])), fabsf(o[2])) > jb->r_safe) {",
     "    if (0) {", "instances: far origins walk the unproven top level (reading A27)"),
    ("oracle.c", "  float x = s * (float)w - 0.5f;\n  float y = t * (float)h - 0.5f;",
     "  float x = s * (float)w;\n  float y = t * (float)h - 0.5f;", "bilinear: texel-centre offset dropped in x"),
    ("oracle.c", "return ((1.0f - fx) * a00 + fx * a10) * (1.0f - fy) + ((1.0f - fx) * a01 + fx * a11) * fy;",
     "return ((1.0f - fx) * a00 + fx * a01) * (1.0f - fy) + ((1.0f - fx) * a10 + fx * a11) * fy;",
     "bilinear: corner texels transposed"),
    ("oracle.c", "long i0 = wrap_long((long)x0, w), i1 = wrap_long((long)x0 + 1, w);",
     "long i0 = (long)x0 < 0 ? 0 : (long)x0 % w, i1 = ((long)x0 + 1) % w;", "bilinear: clamp instead of wrap at the seam"),
    ("oracle.c", "long cs = (long)floorf(coord[0] * fm), ct = (long)floorf(coord[1] * fm);",
     "long cs = (long)floorf(u * fm), ct = (long)floorf(coord[1] * fm);", "uv checker: barycentric u instead of s"),
    ("walker.c", "float a = ((1.0f - fx) * a00 + fx * a10) * (1.0f - fy) + ((1.0f - fx) * a01 + fx * a11) * fy;",
     "float a = ((1.0f - fx) * a00 + fx * a10) * (1.0f - fy) + ((1.0f - fx) * a01 + fx * a11) * fx;",
     "walker bilinear: fx used as the row weight"),
    ("walker.c", "              mbw[pos] = mbw[pos - 1];\n", "",
     "list multi-hit: list index not moved with its hit"),
    ("walker.c", "              S->mbw[pos] = S->mbw[pos - 1];\n", "",
     "instance multi-hit: instance index not moved with its hit"),
    ("walker.c", "            if (S->nk == S->K) S->best_t = S->mb[S->K - 1].t;\n", "",
     "instance multi-hit: a full buffer does not shrink tmax"),
    # ---- slab contract r02 (round 2: tests/test_oracle_slab_r02.py) ----
    ("walker.c", "  *pad = fmaxf(fmaxf(fabsf(e[0]), fabsf(e[1])), fabsf(e[2])) * 4.0f;", "  *pad = 0.0f;",
     "slab r02: no allowance for the fma form's absolute error"),
    ("walker.c", "  tf = fminf(tf, best_t + pad);", "  tf = fminf(tf, best_t);",
     "slab r02: best_t bound without the allowance"),
    ("walker.c", "  float t0x = fmaf(lo[0], inv[0], noi[0]), t1x = fmaf(hi[0], inv[0], noi[0]);",
     "  float t0x = (lo[0] - o[0]) * inv[0], t1x = (hi[0] - o[0]) * inv[0];",
     "slab r02: x planes in the round-1 sub-mul form"),
    ("walker.c", "  for (int a = 0; a < 3; ++a) e[a] = fmaf(o[a], inv[a], noi[a]);",
     "  for (int a = 0; a < 3; ++a) e[a] = o[a] * inv[a] + noi[a];",
     "slab r02: rounding error of noi taken from an unfused sum (always 0)"),
    # ---- ambiguity flags X1-X5 (round 2: tests/test_oracle_flags.py) ----
    ("oracle.c", "(double)second_t - (double)best.t < 1e-5 * fabs((double)best.t))",
     "(double)second_t - (double)best.t < 1e-7 * fabs((double)best.t))", "X1: tie band 100x too narrow"),
    ("oracle.c", "      if (t < second_t) second_t = t;\n", "",
     "X1: a later, farther candidate never becomes the runner-up"),
    ("oracle.c", "second_t = have ? best.t : second_t;", "second_t = second_t;",
     "X1: the displaced best is not kept as the runner-up"),
    ("oracle.c", "if (fabs(m) < 1e-6) f |= OR_X2_EDGE_GRAZE;", "if (m >= 0 && m < 1e-6) f |= OR_X2_EDGE_GRAZE;",
     "X2: only grazes from inside flagged"),
    ("oracle.c", "    m = m < w ? m : w;\n    if (fabs(m)", "    if (fabs(m)",
     "X2: third barycentric (1-u-v) dropped from the margin"),
    ("oracle.c", "if (d0 != d1 || d0 != d2 || d0 != d3) f |= OR_X3_TEXEL_EDGE;", "f |= OR_X3_TEXEL_EDGE;",
     "X3: no straddle check (every texel line flagged)"),
    ("oracle.c", "if (dist_to_int(ss * W) < 1e-5 || dist_to_int(tt * H) < 1e-5) {",
     "if (dist_to_int(ss * W) < 1e-5) {", "X3: row lines (t*H) not checked"),
    ("oracle.c", "if (dist_to_int(u * M) < 1e-6 * M || dist_to_int(v * M) < 1e-6 * M) f |= OR_X4_CHECKER_EDGE;",
     "if (dist_to_int(u * M) < 1e-6 * M) f |= OR_X4_CHECKER_EDGE;", "X4: v cell edges not checked"),
    ("oracle.c", "      double M = (double)jb->M;\n      if (dist_to_int(u * M)",
     "      double M = 8.0;\n      if (dist_to_int(u * M)", "X4: fixed M = 8 instead of the call's frequency"),
    ("oracle.c", "        double band = 1e-6;", "        double band = 1e-8;", "X5: floor below north_star's 1e-6"),
    ("oracle.c", "        double band = 1e-6;", "        double band = 1e-4;", "X5: round-1 blanket 1e-4 band"),
    ("oracle.c", "          band += 2.0 * (W_of(s, k) * fabs((double)st32[0] - ss) +\n"
                 "                         H_of(s, k) * fabs((double)st32[1] - tt));\n", "",
     "X5: fp32 texcoord error not propagated into the band"),
]


def run():
    rows = []
    for fname, orig, mut, desc in MUTANTS:
        tmp = tempfile.mkdtemp(prefix="mut_")
        try:
            for f in ("oracle.c", "walker.c", "oracle.h"):
                shutil.copy(os.path.join(ORACLE, f), tmp)
            path = os.path.join(tmp, fname)
            src = open(path).read()
            if orig not in src:
                rows.append((desc, "NOT APPLIED (snippet not found)", ""))
                continue
            open(path, "w").write(src.replace(orig, mut, 1))
            lib = os.path.join(tmp, "libmut.so")
            b = subprocess.run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
                                "-fno-fast-math", "-pthread", "-D_GNU_SOURCE", "-w", "-o", lib,
                                os.path.join(tmp, "oracle.c"), os.path.join(tmp, "walker.c"), "-lm"],
                               capture_output=True, text=True)
            if b.returncode != 0:
                rows.append((desc, "does not compile", ""))
                continue
            env = dict(os.environ, ORACLE_MUTANT_LIB=lib)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                *PINS], cwd=ROOT, env=env, capture_output=True, text=True,
                               timeout=900)
            failed = [ln.split("::")[-1].split(" ")[0] for ln in r.stdout.splitlines()
                      if ln.startswith("FAILED")]
            status = "killed" if r.returncode != 0 else "SURVIVED"
            rows.append((desc, status, ", ".join(failed[:2])))
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
    return rows


if __name__ == "__main__":
    rows = run()
    print("# r02 — oracle mutation check (CPU pins only)\n")
    print("Each row patches one plausible mistake into a copy of `oracle/*.c`, builds it, and runs")
    print("`" + " ".join(PINS) + "` against it. A pin suite is adequate if every mutant is killed.\n")
    print("| mutant | result | first failing pin |")
    print("|---|---|---|")
    for d, s, f in rows:
        print(f"| {d} | {s} | {f} |")
    killed = sum(1 for _, s, _ in rows if s == "killed")
    print(f"\n{killed} / {len(rows)} mutants killed.")
