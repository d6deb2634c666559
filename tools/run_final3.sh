cd /root/repo
bash tools/run_final.sh
bash tools/run_ncu_final.sh
