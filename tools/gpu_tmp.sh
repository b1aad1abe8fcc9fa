#!/bin/bash
timeout 600 python -m pytest tests/test_api_gpu.py -q -x 2>&1 | tail -5
