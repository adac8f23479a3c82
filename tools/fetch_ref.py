"""Stage the unmodified reference under baseline/_ref (git-ignored, travels to the GPU box).

    python tools/fetch_ref.py          # idempotent; needs /root/reference (build container)

1. `pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse
   --target baseline/_ref <copy of /root/reference/pkg>` -- the reference package
   `ranswitch` exactly as shipped (dependency resolution is skipped: numpy / scipy are
   already in the image; the copy under /tmp because /root/reference is read-only).
2. The reference's own test suite and configs are copied to baseline/_ref/refpkg/
   {tests,configs} (same relative layout, so `test_harness.py`'s `parents[1]/configs`
   resolves) -- the GPU drop-in test runs them with the device path rebound.
Nothing here is committed; the recipe is.  `__graft_entry__.build()` calls it when
/root/reference exists and the staged copy is missing or stale.
"""
from __future__ import annotations

import hashlib
import pathlib
import shutil
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF_PKG = pathlib.Path("/root/reference/pkg")
DEST = ROOT / "baseline" / "_ref"
STAMP = DEST / ".source_sha256"


def source_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(REF_PKG.rglob("*")):
        if p.is_file() and "__pycache__" not in p.parts:
            h.update(str(p.relative_to(REF_PKG)).encode())
            h.update(p.read_bytes())
    return h.hexdigest()


def staged() -> bool:
    return (DEST / "ranswitch" / "__init__.py").exists() and (DEST / "refpkg" / "tests").exists()


def fetch(force: bool = False) -> pathlib.Path:
    if not REF_PKG.exists():
        if staged():
            return DEST
        raise FileNotFoundError(f"{REF_PKG} is not present and {DEST} is not staged")
    digest = source_digest()
    if not force and staged() and STAMP.exists() and STAMP.read_text() == digest:
        return DEST
    if DEST.exists():
        shutil.rmtree(DEST)
    with tempfile.TemporaryDirectory() as tmp:
        src = pathlib.Path(tmp) / "pkg"
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(DEST), str(src),
               "-q"]
        subprocess.run(cmd, check=True)
    for sub in ("tests", "configs"):
        shutil.copytree(REF_PKG / sub, DEST / "refpkg" / sub,
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    STAMP.write_text(digest)
    return DEST


if __name__ == "__main__":
    print(fetch(force="--force" in sys.argv))
