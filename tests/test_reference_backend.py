"""The drop-in boundary proven on the real reference: its own engine tests
(pkg/tests/test_engine.py, all of them) and acceptance criterion 7 (the
6,298,419-candidate sweep with flat memory, test_acceptance.py:273-313) run
UNMODIFIED with `_scan_range` -- the backend seam of engine.py:241 -- and the
worker initializer routed through simba_scan_range
(paper_2605_08243_b200.reference_backend).

The reference package and its tests are installed into baseline/_ref (git-
ignored, shipped to the GPU box with the snapshot; DESIGN.md records the
install command)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
REF_TESTS = REF / "mbasynth_tests"


def _ref_pytest(args, tmp_path, timeout):
    if not (REF / "mbasynth").is_dir() or not REF_TESTS.is_dir():
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md: reference install)")
    launches = tmp_path / "launches.txt"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests")])
    env["SIMBA_REF_LAUNCHES"] = str(launches)
    cmd = [sys.executable, "-m", "pytest", *args, "-p", "ref_backend_plugin", "-p", "no:cacheprovider", "-q",
           "--rootdir", str(REF_TESTS)]
    p = subprocess.run(cmd, cwd=str(REF_TESTS), env=env, capture_output=True, text=True, timeout=timeout)
    tail = (p.stdout + p.stderr)[-4000:]
    return p.returncode, int(launches.read_text()) if launches.exists() else 0, tail


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_reference_engine_tests_through_simba_scan_range(tmp_path):
    rc, launches, tail = _ref_pytest(["test_engine.py"], tmp_path, 800)
    assert rc == 0, tail
    assert launches > 0, "the reference ran without touching libsimba"
    print(tail)


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_reference_criterion_7_through_simba_scan_range(tmp_path):
    rc, launches, tail = _ref_pytest(["test_acceptance.py::test_criterion_7_sweep_throughput_and_flat_memory",
                                      "-rA"], tmp_path, 800)
    assert rc == 0, tail
    assert launches > 0, "the reference ran without touching libsimba"
    print(tail)


def test_backend_install_swaps_only_the_seam():
    """CPU: install() replaces exactly the backend seam of a module shaped like
    the reference's engine and leaves Algorithm 1 alone."""
    from types import SimpleNamespace

    from paper_2605_08243_b200 import reference_backend

    def synthesize():
        pass

    mod = SimpleNamespace(synthesize=synthesize, _EvalContext=object, _scan_range=None, _init_worker=None,
                          _scan_task=None, ProcessPoolExecutor=None)
    reference_backend.install(mod)
    assert mod.synthesize is synthesize
    assert mod._EvalContext is reference_backend.DeviceEvalContext
    assert mod._scan_range is reference_backend.scan_range
    assert mod._init_worker is reference_backend.init_worker
    assert mod._scan_task is reference_backend.scan_task
    assert mod.ProcessPoolExecutor.keywords["mp_context"].get_start_method() == "spawn"
