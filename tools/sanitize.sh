#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over smoke() and the GPU
# tests that reach every kernel: encoders, the trigger kernel's record buffer
# (all-pairs, overflow replay, 8/16-byte records, multi-chunk with and
# without the chunk filter), the radix-select reduce and compaction, the
# record ordering sort, the batched append, clause lookup, multi-shard rounds,
# the host report ring (mapped host memory, bounded waits).
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck; do
  echo "== $tool: smoke"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
done
T="tests/test_gpu_engine.py::test_mixed_staging_encodes_identically tests/test_gpu_engine.py::test_widths_and_multichunk_parity tests/test_gpu_engine.py::test_reduce_and_remove_parity
   tests/test_gpu_engine.py::test_report_buffer_overflow_replay tests/test_gpu_engine.py::test_packed_rows_encode_identically
   tests/test_gpu_engine.py::test_twelve_byte_egress_records tests/test_gpu_engine.py::test_get_clauses_and_counters
   tests/test_gpu_ordering.py tests/test_gpu_exchange.py::test_replay_reference_solver_rounds
   tests/test_gpu_streaming.py::test_streaming_parity_vs_oracle_engine
   tests/test_gpu_ring.py"
echo "== memcheck: kernels of the round, reduce, ordering, streaming, shards"
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest -q -x -m gpu -p no:cacheprovider \
  -k "not 2_000_000" $T 2>&1 | tail -3
echo "== racecheck: shared-memory users (encoder stage, record buffer, sort, compaction)"
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest -q -x -m gpu -p no:cacheprovider \
  "tests/test_gpu_engine.py::test_packed_rows_encode_identically" "tests/test_gpu_engine.py::test_report_buffer_overflow_replay" \
  "tests/test_gpu_engine.py::test_reduce_and_remove_parity" "tests/test_gpu_ordering.py" -k "not 2_000_000" 2>&1 | tail -3
