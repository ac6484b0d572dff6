#!/bin/bash
timeout 120 python tools/r2/sconv_timeline.py 0 $(( (14<<21) | (1<<20) )) 2>&1 | head -8
