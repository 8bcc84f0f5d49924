#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over smoke() and small GPU parity tests
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
done
echo "== memcheck: packed/int8 encode, async rounds, streaming"
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest -q -x -m gpu -p no:cacheprovider \
  "tests/test_gpu_engine.py::test_packed_rows_encode_identically" \
  "tests/test_gpu_engine.py::test_async_rounds_match_sync_rounds" \
  "tests/test_gpu_engine.py::test_report_buffer_overflow_replay" \
  "tests/test_gpu_streaming.py::test_streaming_parity_vs_oracle_engine" 2>&1 | tail -4
echo "== racecheck / memcheck: cp.async encoder, dynamic tiles, egress formats, clause lookup"
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest -q -x -m gpu -p no:cacheprovider \
  "tests/test_gpu_engine.py::test_packed_rows_encode_identically" 2>&1 | tail -3
TSG_DYN_TILES=1 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest -q -x -m gpu -p no:cacheprovider \
  "tests/test_gpu_engine.py::test_twelve_byte_egress_records" \
  "tests/test_gpu_engine.py::test_get_clauses_and_counters" \
  "tests/test_gpu_engine.py::test_timing_sampling" 2>&1 | tail -3
