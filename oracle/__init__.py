"""Parity oracle for the B200 HISA path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product path
(``paper_1810_00845_b200``) never imports it and shares no code with it.

Contents
--------
* ``ckks_oracle.c`` -- plain C RNS-CKKS: textbook NTT, ``(unsigned __int128)a*b % q``,
  ChaCha20 samplers, keys, encode/decode, key switching, rotation, rescale.
* ``ckks.py``      -- ctypes wrapper + HISA-shaped object API with scale/level tracking (A8).
* ``nets.py``      -- the paper's Alg. 1 conv (literal, un-hoisted), activation, pools, FC on
  top of ``ckks.py``; and the float64 plaintext evaluation of the same networks.

Parity status: every function is pinned by ``tests/test_oracle_pins.py`` (see DESIGN.md
"Pins"); the paper's own latency numbers are not reproducible -> "parity unpinned" vs paper.
"""
