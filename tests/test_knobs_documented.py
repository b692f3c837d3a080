"""Every runtime knob the library reads (std::getenv("SF_...") in csrc/) is
documented in INTEGRATION.md's knob table."""
import pathlib
import re

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_every_env_knob_is_documented():
    src = ROOT / "paper_2506_22668_b200" / "csrc"
    names = set()
    for f in list(src.glob("*.cu")) + list(src.glob("*.cpp")) + list(src.glob("*.hpp")) + list(src.glob("*.cuh")):
        names.update(re.findall(r'getenv\("(SF_[A-Z0-9_]+)"\)', f.read_text()))
    doc = (ROOT / "INTEGRATION.md").read_text()
    missing = sorted(n for n in names if f"`{n}`" not in doc)
    assert not missing, f"undocumented knobs: {missing}"
    assert len(names) >= 20
