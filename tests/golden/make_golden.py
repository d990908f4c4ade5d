"""Regenerate tests/golden/golden.json from the UNMODIFIED reference build (TEST
INFRASTRUCTURE; needs /root/reference to build oracle/_ref/libsfref.so):

    make -C oracle ref && python tests/golden/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from tests import golden_cases, oracle_backends  # noqa: E402


def main():
    ref = oracle_backends.reference()
    if ref is None:
        sys.exit("oracle/_ref/libsfref.so is not built (needs /root/reference): make -C oracle ref")
    out = {"generator": "tests/golden/make_golden.py over oracle/_ref/libsfref.so (unmodified reference sources)",
           "cases": {name: fn(ref) for name, fn in golden_cases.CASES.items()}}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
        f.write("\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
