for c in 2 3 4 6 8; do echo "== CTAs/SM $c"; FKV_CTAS_PER_SM=$c python tools/probe_shard.py 2>&1 | grep default; done
