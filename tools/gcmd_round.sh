#!/bin/bash
bash tools/gcmd_verify.sh
bash tools/gcmd_ncu.sh
echo all-done
