cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "parity_small or C5 or pipelined or batch_tile_16 or bt8 or partition or lstm_parity or gru or T0 or smem_weight or C3" > gpurun_out/pf_tests.log 2>&1; echo tests=$? >> gpurun_out/pf_tests.log
TAG=pf ENVS="X=0;SRNN_BT=2;SRNN_BT=2 SRNN_PF=0;SRNN_BT=1" QT=";--B 8;--B 8 --bt 4" bash scripts/env_sweep.sh
TAG=pf5 ENVS="X=0;SRNN_PF=0" QT="--H 5760 --B 64 --d 0.1 --T 64 --reps 3" bash scripts/env_sweep.sh
