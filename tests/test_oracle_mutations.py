"""Mutation check of the oracle's pins (③: "chosen so that a plausible mistake anywhere in it fails
one of them"): each case below plants one plausible mistake in a COPY of oracle/ -- a
dropped term, a wrong sign or index, a transposed operand, an off-by-one -- and runs
tests/test_oracle_pins.py against the mutant. Every mutant must be caught (the pins fail); the
unmutated copy must pass. CPU only, a few seconds per mutant."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, exact source snippet of oracle/kvstream.py, mutated snippet)
MUTANTS = [
    ("region_bytes drops the K+V factor",
     "    return 2 * nL * nR * n * n_heads * head_dim * elem_bytes",
     "    return nL * nR * n * n_heads * head_dim * elem_bytes"),
    ("wire order: heads before requests",
     "    return (((((l - l0) * 2 + kv) * nR + (r - r0)) * nH + (h - h0)) * n + (s - s0)) * head_dim + d",
     "    return (((((l - l0) * 2 + kv) * nH + (h - h0)) * nR + (r - r0)) * n + (s - s0)) * head_dim + d"),
    ("pack stacks K/V outermost instead of under the layer",
     "    wire = np.stack(blocks, axis=1)",
     "    wire = np.stack(blocks, axis=0)"),
    ("route intersection off by one (empty pieces kept)",
     "                            if a < b and c < d and (not tp or e < f):",
     "                            if a <= b and c <= d and (not tp or e < f):"),
    ("route destination offsets accumulated per source block",
     "        p.dst_wire_off = dst_acc.get(kd, 0)\n        dst_acc[kd] = p.dst_wire_off + p.bytes",
     "        p.dst_wire_off = dst_acc.get(ks, 0)\n        dst_acc[ks] = p.dst_wire_off + p.bytes"),
    ("route ignores the destination's layer bounds",
     "                            a = max(l0, src.layer_bounds[i], dst.layer_bounds[j])",
     "                            a = max(l0, src.layer_bounds[i])"),
    ("FT6D key: packet and in-packet index swapped",
     "            return (lp, rp, hp, d // x, s, d % x)",
     "            return (lp, rp, hp, d % x, s, d // x)"),
    ("cache addressing forgets the request offset",
     "        lp, rp, hp = l - self.layer_begin, r - self.req_begin, h - self.head_begin",
     "        lp, rp, hp = l - self.layer_begin, r, h - self.head_begin"),
    ("token step t writes position p+t (reading Q4 violated)",
     "    return prompt_len + step - 1",
     "    return prompt_len + step"),
    ("swap rotation direction reversed",
     "    return (x + 1) % n, (x - 1) % n",
     "    return (x - 1) % n, (x + 1) % n"),
    ("uneven layer split gives the extra layers to the last stages",
     "        b.append(b[-1] + q + (1 if st < rem else 0))",
     "        b.append(b[-1] + q + (1 if st >= n_stages - rem else 0))"),
    ("recovery takes the replica from the predecessor",
     '    return [((x + 1) % n, x, "replica_of_x"), ((x - 1) % n, x, "own_cache_of_prev")]',
     '    return [((x - 1) % n, x, "replica_of_x"), ((x - 1) % n, x, "own_cache_of_prev")]'),
    ("swap-in moves only the newest position",
     "    return i * batch * c_bytes",
     "    return batch * c_bytes"),
    # scenario oracles (oracle/scenarios.py)
    ("swap-out writes the position after the last token",
     "        pos = length[x] - 1\n",
     "        pos = length[x]\n", "scenarios.py"),
    ("swap-in brings back only the newest position",
     "        reg = (L0, L1, host[x].req_begin, host[x].req_begin + host[x].n_reqs, 0, length[x])",
     "        reg = (L0, L1, host[x].req_begin, host[x].req_begin + host[x].n_reqs, length[x] - 1, length[x])",
     "scenarios.py"),
    ("ring replicates into its own store instead of the successor's",
     "        remap(own[x], replica[ring_successor(x, n)], region_of(x))",
     "        remap(own[x], replica[x], region_of(x))", "scenarios.py"),
    ("unpack swaps K and V",
     "        dst.set_logical(kv, l0, l1, r0, r1, s0, s1, w[:, kv], (h0, h1))",
     "        dst.set_logical(kv, l0, l1, r0, r1, s0, s1, w[:, 1 - kv], (h0, h1))"),
    ("route source offsets accumulated per destination block",
     "        p.src_wire_off = src_acc.get(ks, 0)\n        src_acc[ks] = p.src_wire_off + p.bytes",
     "        p.src_wire_off = src_acc.get(kd, 0)\n        src_acc[kd] = p.src_wire_off + p.bytes"),
    ("range check off by one (pos_end == max_seq rejected)",
     "        if s1 > s.max_seq:",
     "        if s1 >= s.max_seq:"),
    ("TP head intersection ignores the destination's head bounds",
     "                                e = max(heads[0], sh[t], dh[v])",
     "                                e = max(heads[0], sh[t])"),
    ("ring successor is the predecessor",
     "    return (x + 1) % n\n\n\ndef recovery_copies",
     "    return (x - 1) % n\n\n\ndef recovery_copies"),
    ("log chunks unpacked without the position shift",
     "        unpack(dst, shifted(first, k * pos_step), log[k * w:(k + 1) * w], mode)",
     "        unpack(dst, first, log[k * w:(k + 1) * w], mode)"),
    ("FT6D packet width fixed at 8 words (wrong for non-16-bit words)",
     "            x = 16 // self.elem_bytes\n            return (lp, rp, hp, d // x, s, d % x)",
     "            x = 8\n            return (lp, rp, hp, d // x, s, d % x)"),
    ("recovery: own cache of the successor instead of the predecessor",
     '((x - 1) % n, x, "own_cache_of_prev")]',
     '((x + 1) % n, x, "own_cache_of_prev")]'),
]


def _tree(tmp, mutant):
    for d in ("oracle", "kvgen"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                        ignore=shutil.ignore_patterns("__pycache__"))
    os.makedirs(os.path.join(tmp, "tests"))
    shutil.copy(os.path.join(ROOT, "tests", "test_oracle_pins.py"), os.path.join(tmp, "tests"))
    shutil.copytree(os.path.join(ROOT, "tests", "golden"), os.path.join(tmp, "tests", "golden"))
    with open(os.path.join(tmp, "tests", "conftest.py"), "w") as f:
        f.write("import json, os, sys\nimport pytest\n"
                "sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))\n"
                "G = os.path.join(os.path.dirname(os.path.abspath(__file__)), 'golden')\n"
                "@pytest.fixture\ndef golden():\n"
                "    return lambda n: json.load(open(os.path.join(G, n)))\n")
    if mutant is not None:
        old, new = mutant[1], mutant[2]
        p = os.path.join(tmp, "oracle", mutant[3] if len(mutant) > 3 else "kvstream.py")
        src = open(p).read()
        assert src.count(old) == 1, f"snippet not found exactly once: {old!r}"
        open(p, "w").write(src.replace(old, new))


def _run(tmp):
    env = dict(os.environ, PYTHONPATH=tmp, PYTHONDONTWRITEBYTECODE="1")
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                           os.path.join(tmp, "tests", "test_oracle_pins.py")],
                          cwd=tmp, env=env, capture_output=True, text=True, timeout=300)


def test_unmutated_copy_passes(tmp_path):
    _tree(str(tmp_path), None)
    r = _run(str(tmp_path))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("mutant", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_pins_catch_mutant(tmp_path, mutant):
    _tree(str(tmp_path), mutant)
    r = _run(str(tmp_path))
    assert r.returncode == 1, f"no pin caught the mutant: {mutant[0]}\n{r.stdout[-1500:]}"
    assert "FAILED tests/test_oracle_pins.py::" in r.stdout   # a pin failed (not a collection error)
