"""Test and benchmark harness (not product code): synthetic BASELINE-config inputs
(`synthetic`) and the config-5 swap-log replay driver (`replay`).  Only tests/,
bench.py, tools/ and __graft_entry__.smoke() import it."""
