"""Mutation check of the oracle pins: each mutation below is a plausible mistake in oracle/oracle.c
(a dropped gate, a flipped sign); applied to a scratch copy of the repo, the CPU pin tests must
FAIL for every one of them.  Prints one line per mutation and exits non-zero if a mutation
survives.
    python tools/mutate_oracle.py"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, exact source text, replacement) -- each text must occur exactly once in oracle.c
MUTATIONS = [
    ("gated: drop the bistatic receive-cone gate",
     "        const double* r = rx + 3 * ((int64_t)p * E + e);\n"
     "        if (bistatic && !in_fov(x, r, a, b, az, el)) continue;\n"
     "        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;\n"
     "        cnt += one_term(",
     "        const double* r = rx + 3 * ((int64_t)p * E + e);\n"
     "        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;\n"
     "        cnt += one_term("),
    ("gated_weighted: drop the transmit-cone gate",
     "      if (!in_fov(x, tx + 3 * p, a, b, az, el)) continue;\n"
     "      const double t0p = t0 ? t0[p] : 0.0;\n"
     "      const double rt = dist3(x, tx + 3 * p);",
     "      const double t0p = t0 ? t0[p] : 0.0;\n"
     "      const double rt = dist3(x, tx + 3 * p);"),
    ("gated_weighted: drop the receive-cone gate",
     "        if (bistatic && !in_fov(x, r, a, b, az, el)) continue;\n"
     "        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;\n"
     "        const double rr = dist3(x, r);",
     "        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;\n"
     "        const double rr = dist3(x, r);"),
    ("gated_motion: gate the receiver at its reception-time position",
     "        if (bistatic && !in_fov(x, r, a, b, az, el)) continue;\n"
     "        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;\n"
     "        const double tau = delay_moving(x, tx + 3 * p, r, vel + 3 * p, c);",
     "        const float* ch = echoes + 2 * ((int64_t)p * E + e) * (int64_t)Ns;\n"
     "        const double tau = delay_moving(x, tx + 3 * p, r, vel + 3 * p, c);\n"
     "        { const double* v = vel + 3 * p; const double rr2[3] = {r[0] + v[0] * tau, r[1] + v[1] * tau, r[2] + v[2] * tau};\n"
     "          if (bistatic && !in_fov(x, rr2, a, b, az, el)) continue; }"),
    ("gated_refracted: drop the transmit-cone gate",
     "      if (!in_fov(x, tx + 3 * p, a, b, az, el)) continue;\n"
     "      const double t0p = t0 ? t0[p] : 0.0;\n"
     "      const double tt = travel_refracted(",
     "      const double t0p = t0 ? t0[p] : 0.0;\n"
     "      const double tt = travel_refracted("),
    ("whitening: periodogram exponent sign flipped",
     "const double a = -TWO_PI * (double)(((int64_t)k * n) % M) / (double)M;",
     "const double a = TWO_PI * (double)(((int64_t)k * n) % M) / (double)M;"),
    ("whitening: imaginary part of the sqrt(G) FIR flipped",
     "      im += sqrt(G[k]) * sin(a);",
     "      im -= sqrt(G[k]) * sin(a);"),
]

MUTATIONS += [
    ("nav: first-order start tangent",
     "      m[i] = 0.5 * (-3.0 * lut[i] + 4.0 * lut[3 + i] - lut[6 + i]);",
     "      m[i] = lut[3 + i] - lut[i];"),
    ("nav: end tangent sign slip",
     "      m[i] = 0.5 * (3.0 * lut[3 * (K - 1) + i] - 4.0 * lut[3 * (K - 2) + i] + lut[3 * (K - 3) + i]);",
     "      m[i] = 0.5 * (3.0 * lut[3 * (K - 1) + i] - 4.0 * lut[3 * (K - 2) + i] - lut[3 * (K - 3) + i]);"),
    ("nav: Hermite basis h10 with (1 - s) once",
     "  const double h10 = s * (1.0 - s) * (1.0 - s);",
     "  const double h10 = s * (1.0 - s);"),
    ("nav: segment index not clamped below (no continued first cubic)",
     "  if (k < 0) k = 0;\n  if (k > K - 2) k = K - 2;\n  s -= (double)k;",
     "  if (k > K - 2) k = K - 2;\n  if (k < 0) { k = 0; s = 0.0; }\n  s -= (double)k;"),
    ("nav: delay evaluated at the transmit-time receiver position (no fixed point)",
     "    nav_eval(lut, K, dt, tau, r);\n    const double nt = (rt + dist3(x, r)) / c;",
     "    const double nt = (rt + dist3(x, r)) / c;"),
    ("gated_nav: drop the receive-cone gate",
     "        if (bistatic && !in_fov(x, rx + 3 * ch, a, b, az, el)) continue;\n"
     "        const float* d = echoes + 2 * ch * (int64_t)Ns;\n"
     "        const double tau = delay_nav(",
     "        const float* d = echoes + 2 * ch * (int64_t)Ns;\n"
     "        const double tau = delay_nav("),
]

TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_next4.py", "tests/test_oracle_gate_pins.py",
         "tests/test_oracle_nav_pins.py"]


def main():
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    survived = 0
    for name, old, new in MUTATIONS:
        n = src.count(old)
        if n != 1:
            print(f"SKIP (pattern found {n} times): {name}")
            survived += 1
            continue
        with tempfile.TemporaryDirectory(prefix="mut_") as d:
            for sub in ("oracle", "synth", "tests"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
            with open(os.path.join(d, "oracle", "oracle.c"), "w") as f:
                f.write(src.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", *TESTS], cwd=d,
                               capture_output=True, text=True)
            killed = r.returncode != 0
            last = (r.stdout.strip().splitlines() or [""])[-1]
            print(f"{'KILLED ' if killed else 'SURVIVED'}  {name}   [{last}]")
            survived += 0 if killed else 1
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
