"""CPU oracle for the Chameleon LoRA-apply hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_2411_17741_b200`) imports this package.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may use it, and only as the checker or the timed CPU baseline, never as the thing
measured or shipped.

Contents and pinning status:
  * lora_ref.py     — numpy restatement of y += (x . A_i) . B_i per segment.  The reference
                      (adaptersim) only models this as a cost term (engine.py:67-77); the
                      paper's arithmetic lived in the un-vendored third-party S-LoRA kernels.
                      Pinned to third-party golden vectors (vLLM 0.22.0 Punica SGMV torch ops,
                      punica_golden.py -> tests/golden/punica_sgmv.npz) and self-checked
                      (linearity, rank-padding, fp64 agreement) in tests/test_oracle.py.
  * punica_golden.py — generates those vectors (run in this container, where vLLM imports).
  * segments_ref.py — numpy restatement of the segment-table builder; pinned against the
                      reference engine's own batch arithmetic (sum of rank * tokens per step,
                      engine.py:64-77) on batches captured from the reference simulate().
  * pool_ref.py     — numpy restatement of the page layout (pack / unpack).
  * gen_golden.py   — regenerates tests/golden/* by importing the reference from
                      /root/reference (decision traces of AdapterCache, captured batches,
                      workload draws, the reference tests' known answers).
"""
