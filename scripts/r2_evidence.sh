#!/bin/bash
# full round-end evidence: tests, smoke, both bench arms, launch lists, ncu captures, config lines
bash scripts/r2_final.sh
bash scripts/r2_configs.sh
