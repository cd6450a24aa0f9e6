#!/bin/bash
for d in ${DBGS:-0 1 2}; do echo "MP_DBG=$d"; MP_DBG=$d python tools/profile_run.py --passes 5 | tail -1; done
