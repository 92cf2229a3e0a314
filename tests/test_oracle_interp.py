"""CPU: the oracle's restatement of SubsampleSpec::row_indices and
InterpOperator::from_spec/apply (proj/src/grid.cpp:91-130,
proj/src/interp.cpp:19-100, 168-186) is bit-identical to the compiled
reference on periodic / non-periodic / boundary-pinned grids of 1-3 axes."""
import numpy as np
import pytest

SPECS = [([24], [3], None), ([24], [5], [1]), ([20, 20], [2, 2], [1, 1]), ([9, 7], [2, 2], None),
         ([9, 7], [4, 4], None), ([9, 7], [3, 2], [1, 0]), ([16, 16, 16], [3, 2, 3], [1, 0, 1]),
         ([12, 10, 8], [3, 3, 3], None), ([10], [4], [1]), ([5, 6], [5, 2], [1, 1]),
         ([32, 32, 32], [2, 2, 2], None), ([32, 32, 32], [4, 4, 4], [1, 1, 1]), ([7], [7], [1])]


@pytest.mark.parametrize("dims,strides,per", SPECS)
def test_interp_port_vs_reference(orc, ref, dims, strides, per):
    J = orc.row_indices(dims, strides, per)
    assert np.array_equal(J, ref.row_indices(dims, strides, per))
    c = orc.seeded_matrix(len(J), 3, 5 + len(J))
    assert np.array_equal(orc.interp_apply(dims, strides, c, per), ref.interp_apply(dims, strides, c, per))


def test_interp_exact_on_multilinear(orc):
    # test_id_core.cpp:394-414: multilinear data is reproduced exactly
    dims = [9, 7]
    x = np.arange(63) % 9
    y = np.arange(63) // 9
    f = 0.3 + 1.7 * x - 0.4 * y + 0.05 * x * y
    for s in (2, 4):
        J = orc.row_indices(dims, [s, s])
        fine = orc.interp_apply(dims, [s, s], f[J][:, None])
        assert np.max(np.abs(fine[:, 0] - f)) <= 1e-12 * np.max(np.abs(f))


def test_extrapolation_required(orc, ref):
    import oracle

    with pytest.raises(oracle.OracleError) as e:
        ref.interp_apply([10], [4], np.ones((3, 1)), None, include_boundary=False)
    assert e.value.name == "ExtrapolationRequired"
    with pytest.raises(oracle.OracleError):
        orc.interp_apply([10], [4], np.ones((3, 1)), None, include_boundary=False)
