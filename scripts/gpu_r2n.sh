#!/bin/bash
# full GPU suite + smoke
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests/ -m gpu -q > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2n_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
