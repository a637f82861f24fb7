"""B200-native (sm_100a) hot path of Baton (arXiv 2410.18701).

* ``baton``     -- ctypes binding of libbaton.so (include/baton.h), same names
* ``scheduler`` -- replicated host-side relay-race planner (no device code)
* ``engine``    -- per-GPU decode loop executing the planner through libbaton
* ``build``     -- nvcc build of libbaton.so for sm_100a

Importing ``baton``/``engine`` loads libbaton.so and fails loudly if it is not
built; there is no CPU fallback.
"""
