# Host-side overhead of one rb_trace call on the tomo bench scene (python wall vs
# library wall vs K1), and per-step value-vs-kernel gaps of the bench.
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python scripts/host_overhead.py tomo 1.0 6
timeout 600 python scripts/host_overhead.py bos 1.0 6
