"""Mutation check of the oracle's pins: copy oracle/, tests/, gen/ to a scratch dir,
apply one plausible mistake at a time to oracle/oracle.c and run the CPU pins
(tests/test_oracle_*.py). Every mutation must turn at least one pin red.

usage: python tools/mutate_oracle.py [scratch_dir]   (prints one line per mutation)
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, [(old, new), ...]) — each replacement must hit exactly once
MUTATIONS = [
    ("O3+O7 R C^p R^T -> R^T C^p R", [
        ("for (int c = 0; c < 3; ++c) s += R[3 * a + c] * Cp[3 * c + b];",
         "for (int c = 0; c < 3; ++c) s += R[3 * c + a] * Cp[3 * c + b];"),
        ("for (int c = 0; c < 3; ++c) s += RC[3 * a + c] * R[3 * b + c];",
         "for (int c = 0; c < 3; ++c) s += RC[3 * a + c] * R[3 * c + b];"),
        ("for (int k = 0; k < 3; ++k) v += R[3 * a + k] * Cp[3 * k + b];",
         "for (int k = 0; k < 3; ++k) v += R[3 * k + a] * Cp[3 * k + b];"),
        ("for (int k = 0; k < 3; ++k) v += RC[3 * a + k] * R[3 * b + k];",
         "for (int k = 0; k < 3; ++k) v += RC[3 * a + k] * R[3 * k + b];"),
    ]),
    ("O3 R C^p R^T -> C^p", [
        ("for (int c = 0; c < 3; ++c) s += RC[3 * a + c] * R[3 * b + c];",
         "for (int c = 0; c < 3; ++c) s += (c == b ? Cp[3 * a + c] : 0.0) + 0.0 * RC[0];"),
    ]),
    ("O3 gate d2 < r2 -> d2 <= r2", [
        ("cj[i] = (best < r2) ? (int32_t)j : -1;", "cj[i] = (best <= r2) ? (int32_t)j : -1;"),
    ]),
    ("O4 gain-ratio denominator x 1/2", [
        ("double rho = (e - en) / den;\n                trace_put",
         "double rho = (e - en) / (0.5 * den);\n                trace_put"),
    ]),
    ("O3 residual sign d = p' - q", [
        ("double d[3] = {q[0] - pp[0], q[1] - pp[1], q[2] - pp[2]};",
         "double d[3] = {pp[0] - q[0], pp[1] - q[1], pp[2] - q[2]};"),
    ]),
    ("O3 Jacobian skew sign", [
        ("    J[0][1] = -pp[2];\n    J[0][2] = pp[1];", "    J[0][1] = pp[2];\n    J[0][2] = -pp[1];"),
    ]),
    ("O1 tie order (d2, -idx)", [
        ("return ((uint64_t)bits << 32) | (uint64_t)(uint32_t)j;",
         "return ((uint64_t)bits << 32) | (uint64_t)(uint32_t)(0x7fffffff - j);"),
    ]),
    ("O2 regularisation (1, eps, 1)", [
        ("            double w[3] = {eps, 1.0, 1.0};", "            double w[3] = {1.0, eps, 1.0};"),
    ]),
    ("O2 eigenvectors read as rows (V^T w V)", [
        ("for (int c = 0; c < 3; ++c) s += V[3 * a + c] * w[c] * V[3 * b + c];",
         "for (int c = 0; c < 3; ++c) s += V[3 * c + a] * w[c] * V[3 * c + b];"),
    ]),
]

CONFTEST = '''import os, sys, pytest
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build(force=True)
    return oracle
'''


def main():
    scratch = sys.argv[1] if len(sys.argv) > 1 else "/tmp/oracle_mutation"
    shutil.rmtree(scratch, ignore_errors=True)
    os.makedirs(scratch)
    for d in ("oracle", "tests", "gen"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(scratch, d),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    with open(os.path.join(scratch, "tests", "conftest.py"), "w") as f:
        f.write(CONFTEST)
    src_path = os.path.join(scratch, "oracle", "oracle.c")
    orig = open(src_path).read()

    def run():
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider"] +
                           sorted(os.path.join("tests", f) for f in os.listdir(os.path.join(scratch, "tests"))
                                  if f.startswith("test_oracle_")),
                           cwd=scratch, capture_output=True, text=True, timeout=1800)
        tail = r.stdout.strip().splitlines()
        failed = [ln.split("::")[-1].split(" ")[0] for ln in tail if ln.startswith("FAILED")]
        return (tail[-1] if tail else r.stderr[-200:]), failed

    summary, _ = run()
    print(f"baseline: {summary}")
    ok = True
    for name, reps in MUTATIONS:
        s = orig
        for old, new in reps:
            if s.count(old) != 1:
                print(f"{name}: pattern not found exactly once: {old[:60]!r}")
                ok = False
                break
            s = s.replace(old, new)
        else:
            with open(src_path, "w") as f:
                f.write(s)
            summary, failed = run()
            killed = "failed" in summary or "error" in summary
            ok &= killed
            print(f"{name}: {'KILLED' if killed else 'SURVIVED'} — {summary}; e.g. {failed[:3]}")
    with open(src_path, "w") as f:
        f.write(orig)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
