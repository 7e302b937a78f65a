# round-2 GPU session recipe: box facts, then the given pytest selection (-s: MEASURED lines)
free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import torch; f,t=torch.cuda.mem_get_info(); print('mem_get_info free', f, 'total', t)"
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -s -p no:cacheprovider > gpurun_out/tests.log 2>&1; echo "tests rc=$?"
grep -E "MEASURED|passed|failed|Error" gpurun_out/tests.log | tail -80
