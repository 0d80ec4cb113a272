"""C-ABI checks that need no GPU: the library loads, exports every symbol include/*.h declares,
and its host-only logic (route planner, byte counts, validation) agrees with the oracle.

The route is independent code on each side (C++ in csrc/route.cpp, numpy loops in oracle/), so
agreement on random setups is a real cross-check; the oracle itself is pinned in
test_oracle_pins.py.
"""
import glob
import os
import random
import re

import pytest

import paper_2403_01876_b200 as dv
from oracle import kvstream as ok

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


PRODUCT_HEADERS = ("dv.h", "dv_trace.h")
TESTING_HEADERS = ("dv_testing.h", "dv_baselines.h")


def declared_symbols(headers=None):
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        if headers is not None and os.path.basename(h) not in headers:
            continue
        for m in re.finditer(r"DV_API\s+[\w\s\*]+?\b(dv[tb]?_\w+)\s*\(", open(h).read()):
            syms.add(m.group(1))
    return syms


def _dynamic_symbols(path):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    return {l.split()[-1] for l in out.splitlines() if " T " in l}


def test_library_exports_every_declared_symbol():
    """libdvstream.so exports exactly the C symbols of dv.h + dv_trace.h (the product); the test
    utilities and prior-art baselines of dv_testing.h / dv_baselines.h live in the separate
    libdvstream_testing.so and are NOT in the product library."""
    L = dv.lib()
    prod, test = declared_symbols(PRODUCT_HEADERS), declared_symbols(TESTING_HEADERS)
    assert declared_symbols() == prod | test and not prod & test
    assert len(prod) >= 30 and len(test) >= 7
    missing = [s for s in prod if not hasattr(L, s)]
    assert not missing, missing
    assert set(dv.exported_symbols()) == prod and set(dv.testing_symbols()) == test
    T = dv.testing_lib()
    assert not [s for s in test if not hasattr(T, s)]
    c_prod = {s for s in _dynamic_symbols(dv.LIB_PATH) if s.startswith(("dv_", "dvt_", "dvb_"))}
    c_test = {s for s in _dynamic_symbols(dv.TESTING_LIB_PATH) if s.startswith(("dv_", "dvt_", "dvb_"))}
    assert c_prod == prod, c_prod ^ prod
    assert c_test == test, c_test ^ test
    assert dv.dv_abi_version() == 4


def test_no_cpu_fallback_without_gpu():
    """dv_create must fail loudly (DV_ECUDA) when no GPU is usable -- never run on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(dv.DVError) as ei:
        dv.dv_create(0)
    assert ei.value.status == dv.DV_ECUDA


def test_partition_validates_before_touching_the_device():
    """dv_partition_create (include/dv.h SM partitions): argument errors are DV_EINVAL before any
    driver call; without a GPU a valid request fails loudly (never a silent no-op)."""
    import torch
    with pytest.raises(dv.DVError) as ei:
        dv.dv_partition_create(0, 0)
    assert ei.value.status == dv.DV_EINVAL
    st = dv.lib().dv_partition_create(0, 8, 0, None, None, None, None, None)
    assert st == dv.DV_EINVAL and "NULL output" in dv.dv_last_error()
    assert dv.lib().dv_partition_destroy(None) == dv.DV_OK
    if not torch.cuda.is_available():
        with pytest.raises(dv.DVError) as ei:
            dv.dv_partition_create(0, 8)
        assert ei.value.status in (dv.DV_ECUDA, dv.DV_ENOTSUP)


def test_oracle_used_only_by_tests_smoke_and_cpu_baseline():
    """The oracle is test infrastructure: the package, kvgen and tools/ never import it, and
    bench.py imports it only inside its CPU-oracle arm (OracleStep: cpu_baseline, --impl reference)."""
    import ast
    import pathlib
    root = pathlib.Path(__file__).resolve().parents[1]

    def oracle_imports(path):
        tree = ast.parse(path.read_text())
        out = []
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            if any(n == "oracle" or n.startswith("oracle.") for n in names):
                out.append(node.lineno)
        return out
    files = [*root.glob("paper_2403_01876_b200/**/*.py"), *root.glob("kvgen/**/*.py"), *root.glob("tools/*.py")]
    assert files
    for f in files:
        assert not oracle_imports(f), f"{f} imports the oracle"
    src = (root / "bench.py").read_text()
    lo = src.index("class OracleStep")
    hi = src.index("\ndef ", src.index("def cpu_baseline"))
    for line in oracle_imports(root / "bench.py"):
        off = sum(len(x) + 1 for x in src.splitlines()[:line - 1])
        assert lo <= off < hi, f"bench.py:{line} imports the oracle outside its CPU-oracle arm"
    for f in root.glob("paper_2403_01876_b200/csrc/*"):
        assert "oracle" not in f.read_text(), f"{f} mentions the oracle"


def test_fast_path_module_builds_and_exports():
    """The CPython fast path (csrc/pyfast.c) is built beside libdvstream.so and exposes the per-call
    entry points; a malformed call raises instead of reaching the library."""
    f = dv.fast()
    assert f is not None and f.__file__.startswith(os.path.dirname(dv.__file__))
    for name in ("scatter", "gather", "remap", "stream_out", "stream_in", "stream_out_direct", "wait", "signal"):
        assert callable(getattr(f, name))
    with pytest.raises(TypeError):
        f.scatter(0, 0)


def _region_bytes_oracle(r, H, D, e):
    return ok.region_bytes(r.layer_begin, r.layer_end, r.req_begin, r.req_end, r.pos_begin, r.pos_end, H, D, e)


def test_region_bytes_matches_spec_example(golden):
    ex = golden("spec_kv_bytes.json")["kv_cache_bytes"][0]
    assert dv.dv_region_bytes(dv.region(0, 12, 0, 1, 0, 1024), 12, 64, 2) == ex["bytes"]
    with pytest.raises(dv.DVError) as ei:
        dv.dv_region_bytes(dv.region(0, 12, 3, 1, 0, 1024), 12, 64, 2)
    assert ei.value.status == dv.DV_EINVAL


def _bounds(rng, lo, hi, k):
    cuts = sorted(rng.sample(range(lo + 1, hi), k - 1)) if k > 1 else []
    return [lo] + cuts + [hi]


FIELDS = ["src_stage", "src_micro", "dst_stage", "dst_micro", "layer_begin", "layer_end", "req_begin",
          "req_end", "pos_begin", "pos_end", "bytes", "src_wire_off", "dst_wire_off"]


@pytest.mark.parametrize("seed", range(200))
def test_route_matches_oracle(seed):
    rng = random.Random(1000 + seed)
    L, R = rng.randint(1, 80), rng.randint(1, 40)
    lo_l, lo_r = rng.randint(0, 3), rng.randint(0, 3)
    sl = _bounds(rng, lo_l, lo_l + L, rng.randint(1, min(L, 8)))
    dl = _bounds(rng, lo_l, lo_l + L, rng.randint(1, min(L, 8)))
    sr = _bounds(rng, lo_r, lo_r + R, rng.randint(1, min(R, 4)))
    dr = _bounds(rng, lo_r, lo_r + R, rng.randint(1, min(R, 4)))
    S1, S2 = rng.randint(1, 4096), rng.randint(1, 4096)
    l0 = rng.randint(lo_l, lo_l + L - 1); l1 = rng.randint(l0 + 1, lo_l + L)
    r0 = rng.randint(lo_r, lo_r + R - 1); r1 = rng.randint(r0 + 1, lo_r + R)
    s0 = rng.randint(0, min(S1, S2) - 1); s1 = rng.randint(s0, min(S1, S2))
    H, D, e = rng.choice([(40, 128, 2), (72, 128, 2), (112, 128, 2), (4, 16, 2), (3, 8, 4)])
    if rng.random() < 0.1:   # sometimes out of range -> both sides must raise the same error
        s1 = max(S1, S2) + 1
    reg = (l0, l1, r0, r1, s0, s1)
    try:
        exp = ok.route(ok.Setup(sl, sr, S1), ok.Setup(dl, dr, S2), reg, H, D, e)
        exp_err = None
    except (ok.MappingError, ok.RangeError, ValueError) as ex:
        exp_err = type(ex)
    if exp_err is not None:
        with pytest.raises(dv.DVError) as ei:
            dv.dv_route(dv.Setup(sl, sr, S1), dv.Setup(dl, dr, S2), dv.region(*reg), H, D, e)
        want = {ok.MappingError: dv.DV_EMAP, ok.RangeError: dv.DV_ERANGE, ValueError: dv.DV_EINVAL}[exp_err]
        assert ei.value.status == want
        return
    got = dv.dv_route(dv.Setup(sl, sr, S1), dv.Setup(dl, dr, S2), dv.region(*reg), H, D, e)
    assert [[getattr(p, f) for f in FIELDS] for p in got] == [[getattr(p, f) for f in FIELDS] for p in exp]


def test_route_c3_and_errors_match_golden(golden):
    g = golden("c3_pieces.json")
    got = dv.dv_route(dv.Setup(g["prompt_layer_bounds"], [0, 8], 1024), dv.Setup(g["token_layer_bounds"], [0, 8], 2048),
                      dv.region(0, 64, 0, 8, 0, 1000), 72, 128, 2)
    assert [[p.src_stage, p.dst_stage, p.layer_begin, p.layer_end] for p in got] == g["pieces"]
    s = dv.Setup([0, 4, 8], [0, 4], 32)
    cases = [
        (dv.Setup([0, 10], [0, 4], 32), s, dv.region(0, 10, 0, 4, 0, 8), dv.DV_EMAP),
        (s, s, dv.region(0, 8, 0, 5, 0, 8), dv.DV_EMAP),
        (s, dv.Setup([0, 8], [0, 4], 16), dv.region(0, 8, 0, 4, 0, 17), dv.DV_ERANGE),
        (dv.Setup([0, 4, 4], [0, 4], 8), s, dv.region(0, 4, 0, 4, 0, 2), dv.DV_EINVAL),
    ]
    for a, b, r, st in cases:
        with pytest.raises(dv.DVError) as ei:
            dv.dv_route(a, b, r, 2, 8, 2)
        assert ei.value.status == st
    with pytest.raises(dv.DVError, match="max_seq 16"):
        dv.dv_route(s, dv.Setup([0, 8], [0, 4], 16), dv.region(0, 8, 0, 4, 0, 17), 2, 8, 2)
    assert dv.dv_route(s, s, dv.region(0, 8, 0, 4, 5, 5), 2, 8, 2) == []


@pytest.mark.parametrize("seed", range(60))
def test_route_with_tp_matches_oracle(seed):
    rng = random.Random(4000 + seed)
    L, R, Hn = rng.randint(1, 30), rng.randint(1, 12), rng.randint(1, 16)
    sl = _bounds(rng, 0, L, rng.randint(1, min(L, 4)))
    dl = _bounds(rng, 0, L, rng.randint(1, min(L, 4)))
    sr = _bounds(rng, 0, R, rng.randint(1, min(R, 3)))
    dr = _bounds(rng, 0, R, rng.randint(1, min(R, 3)))
    sh = _bounds(rng, 0, Hn, rng.randint(1, min(Hn, 4)))
    dh = _bounds(rng, 0, Hn, rng.randint(1, min(Hn, 4)))
    h0 = rng.randint(0, Hn - 1); h1 = rng.randint(h0 + 1, Hn)
    reg = (0, L, 0, R, 2, 9) + ((h0, h1) if rng.random() < 0.5 else (0, 0))
    exp = ok.route(ok.Setup(sl, sr, 16, sh), ok.Setup(dl, dr, 16, dh), reg, Hn, 64, 2)
    got = dv.dv_route(dv.Setup(sl, sr, 16, sh), dv.Setup(dl, dr, 16, dh), dv.region(*reg), Hn, 64, 2)
    F = FIELDS + ["src_tp", "dst_tp", "head_begin", "head_end"]
    assert [[getattr(p, f) for f in F] for p in got] == [[getattr(p, f) for f in F] for p in exp]


def test_c_program_uses_the_abi_route_only():
    """tests/c/abi_smoke.c: the ABI from plain C (gcc, no Python) -- host route + error naming."""
    import subprocess
    exe = os.path.join(ROOT, "tests", "c", "abi_smoke")
    r = subprocess.run([exe, "--route-only"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "route ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_program_streams_through_the_abi():
    import subprocess
    exe = os.path.join(ROOT, "tests", "c", "abi_smoke")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "stream ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_program_streams_on_an_sm_partition():
    """The same C stream check with every call on the streaming stream of an 8-SM partition made
    by dv_partition_create (green contexts), from plain C."""
    import subprocess
    exe = os.path.join(ROOT, "tests", "c", "abi_smoke")
    r = subprocess.run([exe, "--partition"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "stream ok" in r.stdout and "partition ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_program_runs_the_headline_token_steps():
    """The headline workload driven from plain C through the ABI alone (decoupled C2 token steps to
    pinned host, completion by the flags): it runs to the last flag and reports its rate."""
    import json
    import subprocess
    exe = os.path.join(ROOT, "tests", "c", "abi_smoke")
    r = subprocess.run([exe, "--token-bench"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["steps"] == 500 and d["c2_token_steps_from_C_gbs"] > 0


def test_struct_layouts_match_the_c_header(tmp_path):
    """Every public struct of include/dv.h has the same size and field offsets in the Python
    binding (ctypes) as in C (gcc compiles offsetof / sizeof of each field): the binding can only
    marshal what the C ABI declares."""
    import ctypes as C
    import subprocess
    structs = {"dv_cache": dv.dv_cache, "dv_region": dv.dv_region, "dv_setup": dv.dv_setup,
               "dv_piece": dv.dv_piece, "dv_endpoint": dv.dv_endpoint, "dv_config": dv.dv_config,
               "dv_ipc_blob": dv.dv_ipc_blob, "dv_dplan": dv.dv_dplan, "dv_dplan_set": dv.dv_dplan_set}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dv.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} sizeof %zu\\n", sizeof({name}));')
        for f in cls._fields_:
            lines.append(f'  printf("{name} {f[0]} %zu\\n", offsetof({name}, {f[0]}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for line in out:
        if line:
            name, field, val = line.split()
            got[(name, field)] = int(val)
    for name, cls in structs.items():
        assert got[(name, "sizeof")] == C.sizeof(cls), name
        for f in cls._fields_:
            assert got[(name, f[0])] == getattr(cls, f[0]).offset, (name, f[0])


def test_binding_signatures_match_the_c_prototypes():
    """Every function the Python binding declares (ctypes argtypes) takes as many arguments as its
    prototype in include/*.h: the binding cannot drift from the C ABI unnoticed."""
    import re
    protos = {}
    for h in ("dv.h", "dv_trace.h", "dv_testing.h", "dv_baselines.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"DV_API\s+[\w\s\*]+?\b(\w+)\s*\(([^)]*)\)\s*;", text):
            args = m.group(2).strip()
            protos[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    checked = 0
    for name, (_res, argtypes) in dv._SIGS.items():
        assert name in protos, f"{name} is bound but not declared in include/*.h"
        assert len(argtypes) == protos[name], (name, len(argtypes), protos[name])
        checked += 1
    assert checked >= 60
