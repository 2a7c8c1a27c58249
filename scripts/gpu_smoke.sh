mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
