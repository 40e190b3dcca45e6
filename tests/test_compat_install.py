"""install()/uninstall() patch the reference package's hot-path names in the
defining modules and in every importer; no GPU compute.
Runs only where the reference is importable (this build container)."""
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture()
def ref_pkg():
    sys.path.insert(0, REF)
    try:
        import sparse_sampler  # noqa: F401
        yield sparse_sampler
    finally:
        sys.path.remove(REF)


def test_install_patches_definers_and_importers(ref_pkg):
    from paper_2602_08642_b200 import compat
    import sparse_sampler.density as D
    import sparse_sampler.optimize as O
    import sparse_sampler.pyramid as P
    orig = (P.reconstruct_core, O.reconstruct_core, O.allocate, O.estimate, ref_pkg.allocate)
    patched = compat.install()
    try:
        assert ("sparse_sampler.optimize", "reconstruct_backward") in patched
        assert P.reconstruct_core is compat.pyramid.reconstruct_core
        assert O.reconstruct_core is compat.pyramid.reconstruct_core
        assert O.reconstruct_backward is compat.pyramid.reconstruct_backward
        assert O.allocate is compat.density.allocate and D.allocate is compat.density.allocate
        assert O.estimate is compat.estimators.estimate
        assert ref_pkg.allocate is compat.density.allocate
        import sparse_sampler.images as I
        assert I.warp_array is compat.images.warp_array
        assert O.warp_array is compat.images.warp_array and O.warp_backward is compat.images.warp_backward
        assert O.tonemap_array is compat.tonemap.tonemap_array and O.tonemap_backward is compat.tonemap.tonemap_backward
        assert O.spatial_loss is compat.losses.spatial_loss and O.temporal_loss is compat.losses.temporal_loss
        # results are built from the reference's own classes while installed
        assert compat._types.TYPES["DensityMap"] is D.DensityMap
        assert compat.install()  # idempotent
    finally:
        compat.uninstall()
    assert (P.reconstruct_core, O.reconstruct_core, O.allocate, O.estimate, ref_pkg.allocate) == orig
    assert compat._types.TYPES["DensityMap"] is compat._types.DensityMap
    assert not compat.installed()
