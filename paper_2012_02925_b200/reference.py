"""Locate the reference package (`blockflow`) for the control-plane pieces this
package consumes as they are (SURVEY.md §2 marks the CLI's config schema and
parser out of scope): an importable `blockflow`, else the offline install in
`baseline/_ref` (travels with the repo to the GPU box), else the source tree of
the development container.  Nothing on the hot path imports this module."""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def load(name):
    """blockflow.<name>, or ImportError saying where it was looked for."""
    try:
        return importlib.import_module(f"blockflow.{name}")
    except ImportError:
        pass
    for path in CANDIDATES:
        if os.path.isdir(os.path.join(path, "blockflow")):
            if path not in sys.path:
                sys.path.append(path)
            return importlib.import_module(f"blockflow.{name}")
    raise ImportError(f"blockflow.{name}: the reference package is needed for the run-config "
                      f"schema; install it into baseline/_ref (DESIGN.md §5) — looked in "
                      f"{', '.join(CANDIDATES)}")


def available():
    try:
        load("cli")
        return True
    except ImportError:
        return False
