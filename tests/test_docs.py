"""The documents cite evidence files that exist: every profiles/, tests/,
tools/, oracle/, include/ and package path named in DESIGN.md, README.md and
INTEGRATION.md is present in the repository (wildcards: at least one match)."""
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PREFIXES = ("profiles/", "tests/", "tools/", "oracle/", "include/", "paper_2010_04760_b200/")


def _paths(doc):
    text = open(os.path.join(ROOT, doc)).read()
    for m in re.finditer(r"`([^`\s]+)`", text):
        p = m.group(1).rstrip(".,;:")
        if p.startswith(PREFIXES) and "/" in p and not p.endswith("/"):
            yield p.split("::")[0]


def test_cited_files_exist():
    missing = []
    for doc in ("DESIGN.md", "README.md", "INTEGRATION.md"):
        for p in _paths(doc):
            if p.startswith(("oracle/_ref/", "include/hweno/")):
                continue  # built artefact (git-ignored) / the reference's headers
            p = re.sub(r":\d+(-\d+)?(, ?\d+(-\d+)?)*$", "", p)  # file:line
            if p.startswith(("tests/", "tools/")) and p.endswith((".cpp", ".hpp", ".inc")):
                continue  # the reference's proj/tests, proj/tools (cited file:line)
            pat = p.replace("…", "*").replace("...", "*")
            if "*" in pat:
                if not glob.glob(os.path.join(ROOT, pat)):
                    missing.append((doc, p))
            elif not os.path.exists(os.path.join(ROOT, pat)):
                missing.append((doc, p))
    assert not missing, missing
