"""ORACLE -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import anything from here, and only as the checker or the
timed CPU baseline -- never as the product path.

  planner_port.py   pure-Python restatement of the reference planner (pinned)
  layer_oracle.py   numpy fp32 restatement of the FSEP layer step (parity unpinned:
                    the reference ships no layer numerics)
  ref.py            ctypes binding of the reference library itself (oracle/_ref)
  build_ref.sh      compiles /root/reference/proj/src into oracle/_ref (never copied)
"""
