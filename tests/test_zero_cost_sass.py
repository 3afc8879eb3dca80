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


def test_no_packed_fma_contraction(sass):
    """The arithmetic contract forbids FMA contraction.  ptxas fuses a packed
    f32x2 multiply feeding a packed add into FFMA2 even under --fmad=false, so the kernels only
    use packed products whose consumers are not packed adds (slab: sub then mul; MT: FMUL2 then
    scalar sums).  Any FFMA2 in the library would break bit-exact parity."""
    bad = [name for name, ins in sass.items() if any(i.split()[0].lstrip("@!P0123456789 ")
                                                     .startswith("FFMA2") or " FFMA2 " in f" {i} "
                                                     for i in ins)]
    assert not bad, bad[:3]
