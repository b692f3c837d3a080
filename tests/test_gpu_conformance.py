"""GPU: the reference's own unit suites against the C++ drop-in.

oracle/_ref/conformance/shapflow_conformance is built here by
`make -C oracle conformance` (needs /root/reference; the binary travels to
the GPU box): proj/tests/test_sampler.cpp, test_gcn.cpp, test_solver.cpp,
test_pipeline.cpp, test_fidelity.cpp, test_oracle.cpp and test_document.cpp,
unchanged, compiled through the doctest shim in
tests/conformance/ and linked so that plan_sizes, generate_masks,
predict_probs, predict, predict_batched, solve_cgls, solve_direct,
rank_edges, explain_node, auto_samples and node_sampling_seed come from
paper_2506_22668_b200/dropin/shapflow_dropin.cpp (libshapflow_b200 on the
GPU) and everything else from the reference core.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "conformance", "shapflow_conformance")


def test_reference_suites_pass_on_the_dropin():
    if not os.path.exists(BIN):
        pytest.skip("conformance binary not built (needs /root/reference at build time)")
    env = dict(os.environ, SHAPFLOW_B200_DEVICE="0")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900, env=env)
    out = p.stdout + p.stderr
    print(out[-6000:])
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-2000:]
    cases, passed, failed = map(int, m.groups())
    assert cases == 65 and failed == 0 and p.returncode == 0, out[-4000:]


ACC = os.path.join(ROOT, "oracle", "_ref", "conformance", "shapflow_acceptance")


@pytest.mark.slow
def test_reference_acceptance_criteria_on_the_dropin():
    """proj/tests/acceptance.cpp (the reference's 11 acceptance criteria:
    exact-Shapley agreement, sampled accuracy, solver agreement, plan
    allocation, rank balance, worker-layout invariance, ...) over the
    drop-in. Criterion 6 also runs the reference CLI in subprocess workers;
    the CLI is not buildable here (CLI11 absent), so that criterion is
    reported but not required."""
    if not os.path.exists(ACC):
        pytest.skip("acceptance binary not built (needs /root/reference at build time)")
    env = dict(os.environ, SHAPFLOW_B200_DEVICE="0")
    p = subprocess.run([ACC], capture_output=True, text=True, timeout=1800, env=env)
    out = p.stdout + p.stderr
    print(out[-8000:])
    lines = {}
    for ln in out.splitlines():
        m = re.match(r"(PASS|FAIL) criterion (\d+):", ln)  # acceptance.cpp:61-65
        if m:
            lines[int(m.group(2))] = m.group(1)
    assert len(lines) == 11, out[-3000:]
    failed = sorted(c for c, v in lines.items() if v != "PASS" and c != 6)
    assert not failed, out[-4000:]
