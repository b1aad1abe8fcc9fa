#!/bin/bash
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "power_of_two" 2>&1 | tail -5
