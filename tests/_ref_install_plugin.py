"""pytest plugin (test-only): route the reference package's hot path to the
GPU with ``compat.install()`` BEFORE the reference's own test modules are
collected, so their ``from sparse_sampler.x import f`` bindings take the
patched functions (SURVEY.md 4 "what the build reuses", item 1).

Used by tests/test_gpu_reference_suite.py as ``-p tests._ref_install_plugin``;
writes a JSON report (patched names, device calls) to $SSB_REF_SUITE_REPORT.
"""
import json
import os


def pytest_configure(config):
    from paper_2602_08642_b200 import compat
    config._ssb_patched = compat.install()


def pytest_sessionfinish(session, exitstatus):
    from paper_2602_08642_b200 import compat
    from paper_2602_08642_b200.compat import _dev
    out = os.environ.get("SSB_REF_SUITE_REPORT")
    if out:
        with open(out, "w") as f:
            json.dump({"installed": compat.installed(), "precision": _dev.precision(),
                       "device_calls": _dev.device_calls,
                       "patched": sorted({f"{m}.{n}" for m, n in session.config._ssb_patched})}, f)
