"""Copy the reference's own test suite (/root/reference/pkg/tests/*.py,
unmodified) into tests/ref_suite/vendor/ (git-ignored, so no reference
source enters the history; it travels to the GPU box with the working tree
like the built .so files).  Run by __graft_entry__.build() when
/root/reference exists.  The copies run against this package through the
``polarsim`` alias in tests/ref_suite/polarsim/; tests/ref_suite/conftest.py
marks them ``gpu`` and lists the expected failures with their causes."""

import shutil
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parent / "vendor"


def vendor() -> int:
    if not SRC.is_dir():
        return 0
    DST.mkdir(exist_ok=True)
    n = 0
    for f in sorted(SRC.glob("*.py")):
        shutil.copyfile(f, DST / f.name)
        n += 1
    return n


if __name__ == "__main__":
    print(f"vendored {vendor()} files into {DST}")
