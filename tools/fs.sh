rm -f /tmp/fstamps.txt
NUFI_FIELD_STAMPS=/tmp/fstamps.txt python tools/profile_run.py wl2 12 > /dev/null 2>&1; tail -4 /tmp/fstamps.txt
rm -f /tmp/fstamps.txt; NUFI_FIELD_STAMPS=/tmp/fstamps.txt python tools/profile_run.py wl3r 8 > /dev/null 2>&1; tail -3 /tmp/fstamps.txt
