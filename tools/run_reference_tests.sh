#!/usr/bin/env bash
# Run the reference's own test suite (read from /root/reference, copied to a temp dir outside the
# repo) against this package: `matmulkit` and its submodules are aliased to paper_2309_00628_b200.
# Without a GPU the compute tests raise EngineUnavailable (no CPU fallback by design); the rest
# (validation, counters, schedule legality, core utilities) must pass.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg/tests}"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/tests"
python - "$TMP/tests/conftest.py" "$REPO" <<'PY'
import sys
p, repo = sys.argv[1], sys.argv[2]
alias = (f"import sys\nsys.path.insert(0, {repo!r})\nimport paper_2309_00628_b200 as _pk\n"
         "sys.modules['matmulkit'] = _pk\n"
         "for _m in ('core', 'kernels', 'schedules', 'hybrid', 'metrics', 'counters', 'cli'):\n"
         "    sys.modules['matmulkit.' + _m] = __import__('paper_2309_00628_b200.' + _m, fromlist=['x'])\n")
s = open(p).read()
open(p, "w").write(alias + s)
PY
cd "$TMP" && python -m pytest tests -q -p no:cacheprovider --tb=line "${@:2}" | tail -5
