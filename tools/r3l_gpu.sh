#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1500 python tools/partition_ab.py "stream_priority=0;stream_priority=2" 6 2 2>&1 | grep rep | tee $O/r3m_prio_ab.jsonl
