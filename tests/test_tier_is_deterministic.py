"""The default run of every random (hypothesis) test draws the same examples each time: the CPU and
GPU tiers are gates, fresh examples are explored with KRN_FUZZ=<n> (round 2)."""

import glob
import os
import re


def test_every_hypothesis_test_is_derandomized_by_default():
    here = os.path.dirname(os.path.abspath(__file__))
    seen = 0
    for path in sorted(glob.glob(os.path.join(here, "test_*.py"))):
        if path == os.path.abspath(__file__):
            continue
        text = open(path, encoding="utf-8").read()
        for m in re.finditer(r"@settings\((.*?)\)\n\s*@given", text, flags=re.S):
            seen += 1
            assert "derandomize=" in m.group(1), f"{os.path.basename(path)}: {m.group(1)[:80]}"
            assert "database=None" in m.group(1), f"{os.path.basename(path)}: example database in use"
    assert seen >= 5
