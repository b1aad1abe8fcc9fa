#!/bin/bash
timeout 900 python -m pytest tests/test_sigma2v_gpu.py -q -x 2>&1 | tail -25
