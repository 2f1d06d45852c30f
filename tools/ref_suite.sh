#!/usr/bin/env bash
# Run the reference package's OWN test files, unmodified, against the GPU drop-in.
#
#   tools/ref_suite.sh setup            # here (needs /root/reference): copy pkg/tests into
#                                       # baseline/_ref/tests (git-ignored, travels with gpurun,
#                                       # never committed -- same standing as the reference install)
#   tools/ref_suite.sh run [files...]   # anywhere: pytest them with `gala` = tests/ref_shim/gala
#
# The shim maps gala.{backend,matvec,conv,sharing,ring,errors,analytics} onto
# paper_2105_01827_b200 and gala.oracle onto oracle/plain.py (the tests' own checker).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
DST="$ROOT/baseline/_ref/tests"
case "${1:-run}" in
  setup)
    mkdir -p "$DST"
    cp /root/reference/pkg/tests/*.py "$DST/"
    chmod u+w "$DST"/*.py
    ls "$DST"
    ;;
  run)
    shift || true
    files=("$@")
    if [ ${#files[@]} -eq 0 ]; then
      files=(test_backend.py test_matvec.py test_conv.py test_sharing.py test_acceptance.py
             test_ring.py test_analytics.py test_oracle.py)
    fi
    cd "$DST"
    PYTHONPATH="$ROOT/tests/ref_shim:$ROOT:$DST" python -m pytest -p no:cacheprovider -q -rfEs \
      -o addopts="" --rootdir "$DST" "${files[@]}"
    ;;
esac
