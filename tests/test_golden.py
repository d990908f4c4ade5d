"""The C restatement (oracle/liboracle.so) against the frozen reference outputs of
tests/golden/golden.json — pins the oracle without /root/reference (bit-exact: every digest
and scalar equal)."""
import json
import os

import pytest

from tests import golden_cases

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")


def load_golden():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("name", sorted(golden_cases.CASES))
def test_port_matches_golden(port, name):
    got = json.loads(json.dumps(golden_cases.CASES[name](port)))  # tuples -> lists, as stored
    assert got == load_golden()[name]


def test_golden_file_covers_every_case():
    assert set(load_golden()) == set(golden_cases.CASES)
