"""Install the UNMODIFIED reference package (`kilofield`, /root/reference/pkg) into oracle/_ref/ -- TEST INFRASTRUCTURE ONLY.

The reference is pure Python/NumPy, so "building" it is a pip install of its own pyproject:

    python -m pip install --no-index --no-build-isolation --no-deps --target oracle/_ref <copy of /root/reference/pkg>

(from a copy under a temporary directory because /root/reference is read-only and setuptools writes build/ and
*.egg-info next to the sources).  oracle/_ref/ is git-ignored -- no reference source enters this repository's
history -- but not gpurun-ignored, so like the built .so files it travels to the GPU box, where /root/reference does
not exist.  Users: `bench.py --impl reference` / the `cpu_baseline` leg (they time kilofield.surface.render_frame
itself, `kind: "reference"`) and tests/test_ref_install.py (the oracle restatement against the installed reference,
and the reference's own tracer driven through the product's FieldSurface).  The product package never imports it.

`__graft_entry__.build()` calls ensure(); on a machine without /root/reference an existing oracle/_ref is used as is
and a missing one is reported by available() == False (bench.py then falls back to the oracle port, `kind: "port"`).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
TARGET = os.path.join(HERE, "_ref")
REFERENCE_PKG = "/root/reference/pkg"


def available() -> bool:
    return os.path.isfile(os.path.join(TARGET, "kilofield", "surface.py"))


def ensure(force: bool = False) -> bool:
    """Install the reference into oracle/_ref if it is not there yet (or `force`).  Returns available()."""
    if available() and not force:
        return True
    if not os.path.isdir(REFERENCE_PKG):
        return available()
    tmp = tempfile.mkdtemp(prefix="kilofield_src_")
    try:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REFERENCE_PKG, src, ignore=shutil.ignore_patterns("frontend", "node_modules", "__pycache__"))
        if os.path.isdir(TARGET):
            shutil.rmtree(TARGET)
        subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation", "--no-deps",
                        "--disable-pip-version-check", "--find-links", "/opt/wheelhouse", "--target", TARGET, src], check=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    return available()


def import_reference():
    """Import the installed reference's hot-path modules (not `kilofield.cli` / `mesh`: they need scikit-image, which
    this image lacks and the path does not use).  Returns the `kilofield` package."""
    if not available():
        raise ImportError("oracle/_ref is not installed: run `python -m oracle.build_ref` where /root/reference exists")
    if TARGET not in sys.path:
        sys.path.insert(0, TARGET)
    import kilofield  # noqa: F401
    import kilofield.cameras  # noqa: F401
    import kilofield.grid  # noqa: F401
    import kilofield.modelio  # noqa: F401
    import kilofield.pathtrace  # noqa: F401
    import kilofield.surface  # noqa: F401

    return kilofield


if __name__ == "__main__":
    ok = ensure(force="--force" in sys.argv)
    print("oracle/_ref:", "installed" if ok else "unavailable (no /root/reference here)")
    sys.exit(0 if ok else 1)
