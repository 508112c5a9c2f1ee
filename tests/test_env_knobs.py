"""Every TPR_* environment knob the native sources read is documented in the
C ABI header (include/tpr.h), and every tuning key the header lists is
accepted by _native's key table."""

import re

from conftest import ROOT

CSRC = ROOT / "paper_2605_05467_b200" / "csrc"


def _source_knobs():
    names = set()
    for f in list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")):
        names |= set(re.findall(r'"(TPR_[A-Z0-9_]+)"', f.read_text()))
    return names


def test_every_env_knob_is_documented_in_the_header():
    header = (ROOT / "include" / "tpr.h").read_text()
    knobs = _source_knobs()
    assert {"TPR_K31", "TPR_BULK_K1", "TPR_BULK_K31"} <= knobs
    missing = sorted(k for k in knobs if k not in header)
    assert not missing, missing


def test_header_tuning_keys_match_native_table():
    from paper_2605_05467_b200 import _native
    header = (ROOT / "include" / "tpr.h").read_text()
    keys = set(re.findall(r'^ \*   "([a-z0-9_]+)"\s+\[TPR_', header, re.M))
    assert keys == set(_native.TUNING_KEYS), (keys, _native.TUNING_KEYS)
