#!/bin/bash
bash scripts/gpu_check.sh "$1"
bash scripts/gpu_profile.sh "$1"
