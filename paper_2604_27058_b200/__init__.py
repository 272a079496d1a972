"""B200-native shot-sampling engine for the near-Clifford ("Clifft"/framesim) bytecode VM.

Host side: the reference compiler's ``BytecodeProgram`` is serialized
(``program.py``) and executed by hand-written sm_100a CUDA engines behind the C
ABI in ``include/fs_sampler.h`` (``_build/libfs_sampler.so``).  ``runtime``
mirrors the reference ``framesim.runtime`` API (sample / sample_accumulate /
run_shot / ShotState / ShotRecord / ShotError).
"""
from .program import Program, serialize, as_program  # noqa: F401

__version__ = "0.1.0"
