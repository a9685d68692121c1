python tools/phase_profile.py 2000000 2>&1 | tail -14
bash tools/gpu_prof_compress.sh
