"""Mutation check of the oracle pins.

Applies each plausible mistake to a COPY of oracle/model.py and runs
tests/test_oracle_pins.py (plus the older model pins) against it; every mutation must make
at least one pin fail, and the unmutated copy must pass.  Usage: python tools/oracle_mutations.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    "sigma/SiLU swapped between branches": ("return torch.sigmoid(hg) * silu(hc)", "return torch.sigmoid(hc) * silu(hg)"),
    "core LayerNorm dropped": ('hc = layer_norm(fc("core"), P[f"{prefix}.ln_core.g"], P[f"{prefix}.ln_core.b"])',
                               'hc = fc("core")'),
    "gate LayerNorm dropped": ('hg = layer_norm(fc("gate"), P[f"{prefix}.ln_gate.g"], P[f"{prefix}.ln_gate.b"])',
                               'hg = fc("gate")'),
    "hidden SiLU of Fc dropped": ('h1 = silu(x @ P[f"{prefix}.{br}.W1"] + P[f"{prefix}.{br}.b1"])',
                                  'h1 = (x @ P[f"{prefix}.{br}.W1"] + P[f"{prefix}.{br}.b1"])'),
    "e^a moved inside phi": ('m = ea * gated_mlp(x, P, f"atom{t}", cfg.gmlp_hidden)',
                             'm = gated_mlp(torch.cat([v[G.ctr], v[G.nbr], e * ea], dim=1), P, f"atom{t}", cfg.gmlp_hidden)'),
    "e^a dropped": ('m = ea * gated_mlp(x, P, f"atom{t}", cfg.gmlp_hidden)',
                    'm = gated_mlp(x, P, f"atom{t}", cfg.gmlp_hidden)'),
    "one e^b factor dropped": ('q = eb[G.a_b1] * eb[G.a_b2] * gated_mlp', 'q = eb[G.a_b1] * gated_mlp'),
    "e^b of first bond used twice": ('q = eb[G.a_b1] * eb[G.a_b2] * gated_mlp', 'q = eb[G.a_b1] * eb[G.a_b1] * gated_mlp'),
    "atom message summed at the neighbour": ("index_add(0, G.ctr, m)", "index_add(0, G.nbr, m)"),
    "bond message summed at the second bond": ("index_add(0, G.a_b1, q)", "index_add(0, G.a_b2, q)"),
    "energy-head hidden SiLU dropped": ('h = silu(h @ P[f"head_E.W{k}"] + P[f"head_E.b{k}"])',
                                        'h = (h @ P[f"head_E.W{k}"] + P[f"head_E.b{k}"])'),
    "force-head hidden SiLU dropped": ('hf = silu(hf @ P[f"head_F.W{k}"] + P[f"head_F.b{k}"])',
                                       'hf = (hf @ P[f"head_F.W{k}"] + P[f"head_F.b{k}"])'),
    "stress-head hidden SiLU dropped": ('hs = silu(hs @ P[f"head_S.W{k}"] + P[f"head_S.b{k}"])',
                                        'hs = (hs @ P[f"head_S.W{k}"] + P[f"head_S.b{k}"])'),
    "energy-head depth 3 instead of 4": ("for k in range(3):\n        h = silu", "for k in range(2):\n        h = silu"),
    "stress not symmetrised": ("Msym = 0.5 * (M + M.transpose(1, 2))", "Msym = M"),
    "angle update drops the residual": ('return a + gated_mlp(_angle_input(v, e, a, G), P, f"angle{t}", 0)',
                                        'return gated_mlp(_angle_input(v, e, a, G), P, f"angle{t}", 0)'),
}

TESTS = ["tests/test_oracle_pins.py"]


def run(tmp):
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *TESTS], cwd=tmp,
                       capture_output=True, text=True)
    return r.returncode, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]


def main():
    src = open(os.path.join(ROOT, "oracle", "model.py")).read()
    ok = True
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "chg_inputs", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__"))
        rc, last = run(tmp)
        print(f"{'unmutated':45s} rc={rc} {last}")
        ok &= rc == 0
        for name, (old, new) in MUTATIONS.items():
            assert src.count(old) >= 1, f"mutation site not found: {name}"
            with open(os.path.join(tmp, "oracle", "model.py"), "w") as f:
                f.write(src.replace(old, new))
            rc, last = run(tmp)
            caught = rc != 0
            ok &= caught
            print(f"{name:45s} {'CAUGHT' if caught else 'MISSED'}  ({last})")
        with open(os.path.join(tmp, "oracle", "model.py"), "w") as f:
            f.write(src)
    print("all mutations caught" if ok else "SOME MUTATIONS MISSED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
