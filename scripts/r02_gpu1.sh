bash scripts/r02_check.sh
SKIP_TESTS=1 bash scripts/r02_iter.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
