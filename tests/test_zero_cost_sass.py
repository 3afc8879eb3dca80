"""Zero-cost claim, static half ("will incur zero cost if no
custom code was supplied"; :83-89 unused code "is never actually compiled").

The NONE instantiation (the overload without an intersector)
and the DEFAULT instantiation (basic_intersector with no override) must compile
to the same SASS instruction stream.  CPU-only: reads the built .so with
cuobjdump.  The timing half (<= 2 %) is measured by bench.py ("zero_cost")."""
import re
import subprocess

import pytest


@pytest.fixture(scope="module")
def sass():
    from paper_1912_12786_b200 import _build
    lib = _build.build()
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if m:
            funcs[cur].append(m.group(1).strip())
    return funcs


def _find(funcs, q, tag, gen=False):
    """The trace kernel for query q and intersector `tag`; gen: the fused ray-generation
    instantiation (template flag GEN, mangled Lb1)."""
    flag = f"{tag}ELb{int(gen)}ELb0E"   # GEN, then OCC = false (the default-occupancy kernel)
    names = [n for n in funcs if f"trace_kernelILi{q}E" in n and "cost_" not in n and flag in n]
    assert len(names) == 1, names
    return funcs[names[0]]


@pytest.mark.parametrize("gen", [False, True])
@pytest.mark.parametrize("q", [0, 1])
def test_none_and_default_sass_identical(sass, q, gen):
    a = _find(sass, q, "14no_intersector", gen)
    b = _find(sass, q, "19default_intersector", gen)
    assert len(a) > 100
    assert a == b


@pytest.mark.parametrize("q", [0, 1])
def test_intersector_code_only_where_used(sass, q):
    """Texture addressing shows up only in instantiations that use it, and the
    default path has no indirect call (no function pointer)."""
    default = _find(sass, q, "19default_intersector")
    alpha = _find(sass, q, "25alpha_texture_intersector")
    fnptr = _find(sass, q, "25runtime_fnptr_intersector")
    # the alpha listing adds sidecar, descriptor and texel loads
    # the byte load of the A8 alpha plane (tex2D) exists only where the alpha
    # intersector is compiled in
    texel = re.compile(r"^(@!?P\d\s+)?LDG\.E\.U8\b")
    assert any(texel.match(i) for i in alpha)
    assert not any(texel.match(i) for i in default)
    indirect = re.compile(r"^(@!?P\d\s+)?CALL\S*\s+R\d+")   # call through a register = fn pointer
    assert not any(indirect.match(i) for i in default)
    assert not any(indirect.match(i) for i in alpha)
    assert any(indirect.match(i) for i in fnptr)


@pytest.fixture(scope="module")
def trace_ptx(tmp_path_factory):
    """PTX of trace.cu (the library embeds SASS only), built with the library's flags."""
    import os
    from paper_1912_12786_b200 import _build
    out = str(tmp_path_factory.mktemp("ptx") / "trace.ptx")
    cmd = [_build.nvcc(), "-O3", "-std=c++17", *_build.ARCH, "-fmad=false", "-prec-div=true",
           "-prec-sqrt=true", "-ftz=false", "-I", os.path.join(_build.ROOT, "include"), "-ptx",
           "-o", out, os.path.join(_build.CSRC, "trace.cu")]
    subprocess.run(cmd, check=True, capture_output=True)
    return open(out).read()


def test_no_packed_fma_contraction(trace_ptx):
    """The arithmetic contract forbids IMPLICIT FMA contraction.  The slab
    test's fused multiply-adds are explicit (contract r02: t = fma(plane, inv, noi) and
    tf = fma(tf, 1 + 2 gamma_3, pad), `fma.rn.f32x2` in the PTX).  ptxas fuses a packed
    f32x2 multiply whose result feeds a packed add/sub into FFMA2 even under --fmad=false,
    so no `mul.rn.f32x2` result may be an operand of an `add`/`sub.rn.f32x2` (MT's packed
    products feed scalar sums); that dataflow is checked on the PTX of every kernel."""
    prods, bad = set(), []
    for line in trace_ptx.splitlines():
        t = line.strip()
        if ".entry " in t or ".func " in t:
            prods = set()
        m = re.match(r"mul\.rn\.f32x2\s+(%rd\d+)", t)
        if m:
            prods.add(m.group(1))
            continue
        m = re.match(r"(add|sub)\.rn\.f32x2\s+%rd\d+,\s*(%rd\d+),\s*(%rd\d+)", t)
        if m and (m.group(2) in prods or m.group(3) in prods):
            bad.append(t)
    assert "fma.rn.f32x2" in trace_ptx
    assert not bad, bad[:3]


def test_slab_uses_explicit_fma(sass):
    """Contract r02: the pair-node slab is FFMA2 (one rounding per plane), not FADD2+FMUL2."""
    body = _find(sass, 1, "19default_intersector")
    assert sum(1 for i in body if "FFMA2" in i) >= 7
