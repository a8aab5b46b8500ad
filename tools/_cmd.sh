python tools/probe_floor.py
echo "--- no PDL"; FKV_NO_PDL=1 python tools/probe_floor.py
echo "--- coop"; FKV_K4_SCHEDULE=coop python tools/probe_floor.py
