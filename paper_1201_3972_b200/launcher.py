"""`python -m paper_1201_3972_b200 ...`: the reference's own command line on the GPU filter.

The reference CLI (irdenoise.cli, cli.py:177-253: add-noise / filter / bench / synth,
its options, messages and exit codes) is used unmodified; `reference_shim.install`
re-points its run_filter at the C ABI before the CLI module binds it. The reference
package is imported from the environment, or from baseline/_ref (the unmodified
reference pip-installed beside this repository).
"""

from __future__ import annotations

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def import_reference():
    """The installed reference package `irdenoise` (ImportError if it is nowhere)."""
    try:
        import irdenoise
    except ImportError:
        ref = os.path.join(REPO, "baseline", "_ref")
        if not os.path.isdir(os.path.join(ref, "irdenoise")):
            raise
        sys.path.insert(0, ref)
        import irdenoise
    return irdenoise


def main(argv=None) -> int:
    ird = import_reference()
    from .reference_shim import install

    install(ird)
    import importlib

    cli = importlib.import_module(ird.__name__ + ".cli")
    install(ird)  # patches the CLI's own binding too
    return cli.main(argv)
