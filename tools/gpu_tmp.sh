#!/bin/bash
timeout 600 python -m pytest tests/test_edge_gpu.py -q -x 2>&1 | tail -25
