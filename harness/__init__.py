"""Bench/test harness: turns a synth.Workload into libblend calls (via the binding)
and device buffers (torch).  Used by bench.py, tests and __graft_entry__.smoke()."""
