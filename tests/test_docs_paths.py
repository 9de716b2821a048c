"""Every profiles/ path that DESIGN.md, README.md and profiles/README.md cite exists (the numbers in
the docs are traceable to a committed file).  CPU only."""
import os
import re

from conftest import ROOT


def test_cited_profile_paths_exist():
    txt = ""
    for f in ("DESIGN.md", "README.md", os.path.join("profiles", "README.md")):
        with open(os.path.join(ROOT, f)) as fh:
            txt += fh.read()
    refs = set(re.findall(r"`(profiles/[A-Za-z0-9_./-]+)`", txt))
    refs |= {"profiles/" + m for m in re.findall(r"`((?:r[12][a-z0-9_]*)/[A-Za-z0-9_./-]*)`", txt)}
    assert len(refs) > 20
    missing = sorted(r for r in refs if not os.path.exists(os.path.join(ROOT, r.rstrip("/"))))
    assert not missing, missing
