"""``python -m paper_2310_19295_b200 <memplan CLI arguments>``

The reference's own command line (``memplan {plan,eval,gen,compare,viz}``,
cli.py:52-96, 319-343; same flags, outputs and exit codes) with the B200 hot
path installed (memplan_plugin.install)."""

from __future__ import annotations

import sys

from . import memplan_plugin


def main(argv: list[str] | None = None) -> int:
    mp = memplan_plugin.install()
    import importlib
    cli = importlib.import_module(mp.__name__ + ".cli")
    return cli.run(argv)


if __name__ == "__main__":
    sys.exit(main())
