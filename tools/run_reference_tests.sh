#!/bin/bash
# Run the reference package's OWN unit tests against this package (drop-in check).
#
# Builds a throwaway import shim in /tmp that maps minhashlab.{families,modmath,corpus,
# minhash} onto paper_1401_6124_b200 (minhashlab.stats, out of scope here, is the
# reference's own module loaded from /root/reference), then runs the reference's tests
# where they lie.  Nothing from /root/reference is copied into this repository.
# Build container only (the GPU box has no /root/reference); signature() needs a GPU,
# so on a CPU-only host test_minhash.py's signature tests fail with "no NVIDIA driver".
# usage: tools/run_reference_tests.sh [pytest args...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=/root/reference/pkg
SHIM=$(mktemp -d /tmp/mhb_shim.XXXX)
mkdir -p "$SHIM/minhashlab"
echo "from paper_1401_6124_b200 import *  # noqa" > "$SHIM/minhashlab/__init__.py"
for m in families modmath corpus minhash; do
  cat > "$SHIM/minhashlab/$m.py" <<PY
from paper_1401_6124_b200 import $m as _m
globals().update({k: getattr(_m, k) for k in dir(_m) if not k.startswith('__')})
PY
done
cat > "$SHIM/minhashlab/stats.py" <<'PY'
import importlib.util as _u, sys as _s
_spec = _u.spec_from_file_location("minhashlab._ref_stats", "/root/reference/pkg/src/minhashlab/stats.py")
_mod = _u.module_from_spec(_spec); _mod.__package__ = "minhashlab"
_s.modules["minhashlab._ref_stats"] = _mod
_spec.loader.exec_module(_mod)
globals().update({k: getattr(_mod, k) for k in dir(_mod) if not k.startswith('__')})
PY
if [ $# -eq 0 ]; then
  set -- "$REF/tests/test_families.py" "$REF/tests/test_modmath.py" "$REF/tests/test_corpus.py" "$REF/tests/test_minhash.py"
fi
cd /tmp
PYTHONPATH="$SHIM:$ROOT" python -m pytest -q -p no:cacheprovider "$@"
