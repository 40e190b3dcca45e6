"""Product-path hygiene: the package never imports the oracle (test-only
checker) and the ops fail loudly without the CUDA library/device."""
import ast
import glob
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_package_never_imports_oracle():
    for path in glob.glob(os.path.join(ROOT, "paper_2602_08642_b200", "**", "*.py"), recursive=True):
        tree = ast.parse(open(path).read())
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            for n in names:
                assert not n.startswith("oracle"), f"{path} imports {n}"


def test_ops_refuse_cpu_tensors():
    torch = pytest.importorskip("torch")
    from paper_2602_08642_b200 import ops
    x = torch.zeros(1, 3, 8, 8)
    with pytest.raises(ValueError):
        ops.pyramid_forward(x, [torch.zeros(1, 29, 8, 8)] * 1)


def test_package_never_reads_staged_reference():
    """baseline/_ref (the staged reference + its tests) is a test-only fixture:
    the product package never names it (compat.install() patches whatever
    `sparse_sampler` the caller has importable)."""
    for path in glob.glob(os.path.join(ROOT, "paper_2602_08642_b200", "**", "*.py"), recursive=True):
        src = open(path).read()
        for needle in ("baseline/_ref", "ref_tests", "/root/reference"):
            assert needle not in src, f"{path} names {needle}"
