"""The reference's simulator CLI (`chunkstar run/sweep/explain-plan/oracle`,
`/root/reference/pkg/src/chunkstar/cli.py`) is OUT OF SCOPE here: it is UX
around the feasibility simulator, not the training step.  The entry point
exists so that drop-in imports resolve; it exits with status 2."""

import sys


def main(argv=None) -> int:
    sys.stderr.write("chunkstar CLI is not part of the B200 chunk-step build; "
                     "use bench.py / paper_2108_05818_b200.trainer\n")
    return 2
