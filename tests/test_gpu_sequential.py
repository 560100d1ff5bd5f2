"""The sequential comparison engine (integrate_sequential, sequential.cpp:45-139;
SURVEY.md 8(f)4) on the GPU against the unmodified reference: bit-identical
estimate, error, status, step count, regions and evaluations."""
import pytest

from ref_ctypes import make_config  # noqa: F401  (conftest puts oracle/ on the path)

pytestmark = pytest.mark.gpu

CASES = [  # fid, n, tau, max_evals, bounds
    (1, 2, 1e-7, 10_000_000, None),
    (3, 5, 1e-5, 2_000_000, None),
    (5, 4, 1e-5, 10_000_000, None),
    (6, 3, 1e-4, 10_000_000, None),
    (4, 8, 1e-3, 10_000_000, None),            # exhausts the evaluation budget
    (2, 6, 1e-3, 10_000_000, None),
    (4, 3, 1e-5, 10_000_000, ([-1.0, 0.0, 0.25], [1.0, 2.0, 0.75])),  # mapped domain
]


@pytest.mark.parametrize("fid,n,tau,max_evals,bounds", CASES)
def test_sequential_matches_reference(pg, gpu, ref, fid, n, tau, max_evals, bounds):
    b = pg.Bounds(*bounds) if bounds else pg.Bounds.unit_cube(n)
    got = pg.integrate_sequential(pg.Integrand(fid), b, tau, max_evals=max_evals)
    want = ref.integrate_sequential(fid, n, tau, max_evals=max_evals,
                                    lower=b.lower if bounds else None,
                                    upper=b.upper if bounds else None)
    assert (got.estimate, got.errorest, str(got.status), got.iterations, got.regions_generated,
            got.eval_count) == (want.estimate, want.errorest, want.status, want.iterations,
                                want.regions_generated, want.eval_count)


def test_sequential_validate_invariants_and_errors(pg, gpu, ref):
    a = pg.integrate_sequential(pg.Integrand(5), pg.Bounds.unit_cube(4), 1e-5,
                                validate_invariants=True)
    b = ref.integrate_sequential(5, 4, 1e-5)
    assert (a.estimate, a.iterations) == (b.estimate, b.iterations)
    with pytest.raises(ValueError):
        pg.integrate_sequential(pg.Integrand(4), pg.Bounds.unit_cube(3), 0.0)
