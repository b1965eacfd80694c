python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/m_build.log 2>&1 || { tail -20 gpurun_out/m_build.log; exit 1; }
tail -1 gpurun_out/m_build.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/m_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/m_pytest.log
