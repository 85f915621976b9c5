timeout 600 tools/shim_timing
