"""FEM assembly as K1 row sums on the device against
the reference's own build_assembly_map + assemble_spmv (fem/assembly.cpp,
compiled from its sources into oracle/_ref): pattern identical, tangent and
residual bitwise (same addends in the same element-major order)."""
import numpy as np
import pytest

from tests.gpu_helpers import bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,ws", [((2, 2, 2), 32), ((4, 3, 5), 32), ((4, 3, 5), 4), ((9, 7, 6), 8)])
def test_assembly_matches_reference(ew, F, dims, ws):
    elems, nnodes = F.box_elements(*dims)
    ne = elems.shape[0]
    rng = np.random.default_rng(ne)
    ke = rng.standard_normal((ne, 16))
    re = rng.standard_normal((ne, 4))
    ro_r, ci_r, t_r, r_r = F.box_assemble(*dims, ke, re, warp_size=ws)
    asm = ew.Assembly(elems, nnodes, warp_size=ws)
    ro, ci = asm.pattern()
    assert np.array_equal(ro, ro_r) and np.array_equal(ci, ci_r)
    t, r = asm.run(ke, re)
    assert np.array_equal(bits(t), bits(t_r))
    assert np.array_equal(bits(r), bits(r_r))


def test_assembly_into_prepared_kernel(ew, F):
    """The tangent assembled straight into a prepared kernel's slots equals
    preparing the kernel on the assembled CSR (the paper's bypass of the
    per-Newton reorder)."""
    elems, nnodes = F.box_elements(5, 4, 3)
    ne = elems.shape[0]
    rng = np.random.default_rng(7)
    ke = rng.standard_normal((ne, 16))
    re = rng.standard_normal((ne, 4))
    asm = ew.Assembly(elems, nnodes)
    ro, ci = asm.pattern()
    t, r = asm.run(ke, re)
    x = rng.uniform(0.1, 1.0, nnodes)
    zeros = ew.Csr(nnodes, nnodes, ro, ci, np.zeros(ci.size))
    filled = ew.Csr(nnodes, nnodes, ro, ci, t)
    for kid in ("k1", "k1rs", "k2"):
        k = ew.Kernel(kid, zeros, threshold=4)
        r2 = asm.run_into(ke, re, k)
        assert np.array_equal(bits(r2), bits(r))
        want = ew.Kernel(kid, filled, threshold=4)
        assert np.array_equal(bits(k.apply(x)), bits(want.apply(x))), kid
    with pytest.raises(ValueError):
        asm.run_into(ke, re, ew.Kernel("csr_ref", zeros))


def test_assembly_errors(ew):
    with pytest.raises(ValueError):
        ew.Assembly(np.array([[0, 1, 2, 9]]), 4)
