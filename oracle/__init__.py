"""Oracle: plain, slow, obviously-correct CPU reference for the blended-batch
tree attention hot path (arXiv 2411.16102, BlendServe).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()`,
`bench.py`'s cpu_baseline / `--impl reference` legs and the committed scripts that
write stored expected values (`scripts/solve_c4_counts.py`) may import anything here.
The product path (`paper_2411_16102_b200`, `libblend.so`) never imports,
links or executes this package, and this package never imports the product.
The two share no code; both draw inputs from `synth/` (input generation only).

Modules
  attention  fp64 softmax(QK^T/sqrt(D))V per request over its materialised path
  tree       descriptor oracle: trie, density keys, Alg-1 sort, DFS ids, pages, classes
  shard      shard oracle: 2G-block fold of the DFS request order
"""
