timeout 1200 python -m pytest tests/test_gpu_bound.py -m gpu -q > gpurun_out/r2cy.log 2>&1; tail -2 gpurun_out/r2cy.log
