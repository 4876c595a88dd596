"""Mutation check of the oracle pins (run by hand: python tests/mutants.py).

Each mutant is a plausible mistake in oracle/hip_oracle.c (a dropped term, a wrong index, a flipped
rule).  The pin suite (tests/test_oracle_pins.py) must fail on every one of them."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "hip_oracle.c")

MUTANTS = {
    "representative = last block of the branch": ("int64_t r = cand[c].f;", "int64_t r = cand[c].l;"),
    "tie-break toward larger block": ("if (a->f < b->f) return -1;\n    if (a->f > b->f) return 1;",
                                      "if (a->f > b->f) return -1;\n    if (a->f < b->f) return 1;"),
    "no causal mask inside the tile": ("if (causal && s > t + delta) continue;\n            const float *kk",
                                       "const float *kk"),
    "tile max over the first query row only": ("int64_t t = t0 + gt % (t1 - t0);", "int64_t t = t0;"),
    "causal bound off by one block": ("int64_t v = (tlast + (Tk - Tq)) / bk + 1;", "int64_t v = (tlast + (Tk - Tq)) / bk;"),
    "initial partition rounds down": ("int64_t fj = lo + (2 * (int64_t)j * L + n) / (2 * (int64_t)n);",
                                      "int64_t fj = lo + (2 * (int64_t)j * L) / (2 * (int64_t)n);"),
    "chunk boundaries round down": ("int64_t a0 = (2 * (int64_t)c * Bq + chunks) / (2 * (int64_t)chunks);",
                                    "int64_t a0 = (2 * (int64_t)c * Bq) / (2 * (int64_t)chunks);"),
    "chunk nodes start at block 0": ("int64_t fj = lo + (2", "int64_t fj = 0 + (2"),
    "keep bottom-n": ("if (a->s > b->s) return -1;\n    if (a->s < b->s) return 1;",
                      "if (a->s < b->s) return -1;\n    if (a->s > b->s) return 1;"),
    "attention drops the max subtraction": ("double p = exp(x[i] - M);", "double p = exp(x[i]);"),
    "attention forgets the softmax scale": ("x[i] = sm_scale * acc;", "x[i] = acc;"),
    # (Bq < n instead of Bq <= n is an EQUIVALENT mutant: with B_q == n every initial node is one
    #  block, the loop never splits and the output is again 0..n-1.)
    "exact case up to 2n": ("if (Bq <= n) { /* exact case */", "if (Bq <= 2 * n) { /* exact case */"),
    "split rounds half down": ("int64_t m = (f + l + 1) / 2;", "int64_t m = (f + l) / 2;"),
    "paged slot uses page index": ("+ s % ps) * d;", "+ s / ps % ps) * d;"),
    "window one token too long": ("for (int64_t s = p - window + 1; s <= p; ++s)", "for (int64_t s = p - window; s <= p; ++s)"),
    "sink ignores causality": ("for (int64_t s = 0; s < imin64(sink, Tk); ++s)\n                    if (!causal || s <= p) tok[ntok++] = s;",
                               "for (int64_t s = 0; s < imin64(sink, Tk); ++s)\n                    tok[ntok++] = s;"),
    "top-r reduces |q| over the first row only": ("for (int64_t t = t0; t < t1; ++t) {\n                double v = fabs(",
                                                 "for (int64_t t = t0; t < t0 + 1; ++t) {\n                double v = fabs("),
    "top-r ties toward the larger component": ("if (!taken[c] && (best < 0 || a[c] > a[best])) best = c;",
                                               "if (!taken[c] && (best < 0 || a[c] >= a[best])) best = c;"),
    "top-r score ignores the component list": ("int c = comp ? comp[i] : i;\n                    acc = fmaf(q[c], kk[c], acc);",
                                               "int c = i;\n                    acc = fmaf(q[c], kk[c], acc);"),
    "jitter range one short": ("% (uint64_t)(2 * R + 1)) - R;", "% (uint64_t)(2 * R)) - R;"),
    "jitter clamp allows an empty left branch": ("if (m < f + 1) m = f + 1;", "if (m < f) m = f;"),
    "vote truncation prefers larger blocks": ("return (a->j > b->j) - (a->j < b->j);\n}\n\nstatic int i32_cmp",
                                              "return (a->j < b->j) - (a->j > b->j);\n}\n\nstatic int i32_cmp"),
    "vote threshold strict": ("if (j - i >= theta)", "if (j - i > theta)"),
    "GQA-shared tile over the first head only": ("for (int64_t gt = 0; gt < (int64_t)G * (t1 - t0); ++gt) {",
                                                 "for (int64_t gt = 0; gt < (int64_t)1 * (t1 - t0); ++gt) {"),
    "GQA-shared rows taken from consecutive heads' wrong rows": ("const float *q = Qh + (gt / (t1 - t0)) * hstride + t * d;",
                                                                  "const float *q = Qh + (gt / (t1 - t0)) * d + t * d;"),
    "F32L tree reversed (o = 1, 2, 4, 8)": ("for (int o = 8; o >= 1; o >>= 1) {", "for (int o = 1; o <= 8; o <<= 1) {"),
    "F32L strided segments instead of contiguous": ("seg[c / w] = fmaf(q[c], kk[c], seg[c / w]);",
                                                    "seg[c % 16] = fmaf(q[c], kk[c], seg[c % 16]);"),
    "F32C accumulates in reverse order": ("for (int i = 0; i < ncomp; ++i) {\n                    int c = comp ? comp[i] : i;\n                    acc = fmaf(",
                                          "for (int i = ncomp - 1; i >= 0; --i) {\n                    int c = comp ? comp[i] : i;\n                    acc = fmaf("),
    "union keeps duplicates": ("if (w == 0 || tok[i] != tok[w - 1]) tok[w++] = tok[i];", "tok[w++] = tok[i];"),
}


def main():
    src = open(SRC).read()
    os.makedirs("/tmp/mut", exist_ok=True)
    survived = []
    for name, (a, b) in MUTANTS.items():
        assert a in src, name
        path = f"/tmp/mut/{abs(hash(name))}.c"
        open(path, "w").write(src.replace(a, b, 1))
        lib = path[:-2] + ".so"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", lib, path, "-lm"])
        env = dict(os.environ, HIP_ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                           env=env, capture_output=True, text=True, cwd=ROOT)
        killed = r.returncode != 0
        print(f"{'KILLED ' if killed else 'SURVIVED'}  {name}")
        if not killed:
            survived.append(name)
    print("survivors:", survived)
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
