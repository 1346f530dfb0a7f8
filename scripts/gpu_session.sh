# scratch driver for one gpurun call; the round-end measurement is scripts/final_measure.sh
bash scripts/final_measure.sh
