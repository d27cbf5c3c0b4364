"""TEST INFRASTRUCTURE - CPU oracle for the B200 execution path.

Restates the reference's algorithm for the hot path on the CPU:

* ``interp``     plain sequential Python/numpy interpreter of any kernel-language
                 function (small sizes)
* ``cport``      ctypes front of ``krn_oracle.c``: the headline objective and the
                 bulk builtins in plain C, usable at full sizes
* ``make_golden`` the script that ran the *reference itself* in the build
                 container and wrote ``tests/golden/`` (needs /root/reference;
                 not runnable on the GPU box)

Parity status: PINNED (see each module's header).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs
may import this package - as the checker, never as the thing measured or
shipped.  ``paper_2507_13204_b200`` does not import it.
"""
