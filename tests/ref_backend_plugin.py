"""pytest plugin (``-p ref_backend_plugin``) for running the UNMODIFIED
reference's own test files with its search routed through libsimba
(paper_2605_08243_b200.reference_backend.install).  Used by
tests/test_reference_backend.py in a subprocess; writes the number of
libsimba kernel launches of the test process to $SIMBA_REF_LAUNCHES."""

import os


def pytest_configure(config):
    import mbasynth.engine as engine

    from paper_2605_08243_b200 import reference_backend

    reference_backend.install(engine)


def pytest_unconfigure(config):
    path = os.environ.get("SIMBA_REF_LAUNCHES")
    if path:
        from paper_2605_08243_b200 import _native as N

        with open(path, "w") as fh:
            fh.write(str(N.launch_count()))
