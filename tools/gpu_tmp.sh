#!/bin/bash
timeout 60 ./tools/tcbench
