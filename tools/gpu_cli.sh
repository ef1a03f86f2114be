timeout 600 python -m pytest tests/test_cli.py -x -q 2>&1 | tail -3
timeout 900 python -m paper_2605_08314_b200 graph-ablation --preset llama7b --rho 0.6 --prompt-len 512 --gen 64 --runs 3 --json gpurun_out/graph_ablation.json 2>&1 | tail -4
