mkdir -p gpurun_out
for c in 1 0; do echo "== cluster=$c"; FK_UPDATE_CLUSTER=$c timeout 300 python scripts/update_small.py; done > gpurun_out/ab_cluster.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_update_cluster -c 20 --csv --log-file gpurun_out/cluster_launches.csv python scripts/update_small.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_update_cluster -s 40 -c 1 -o gpurun_out/cluster_f16 -f python scripts/update_small.py > /dev/null 2>&1
