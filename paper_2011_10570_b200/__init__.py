"""B200-native LTS/GTS octree wave solver (drop-in for the ``amrlts`` API).

Modules mirror the reference package: ``octree``, ``partition``, ``mesh``,
``wave``, ``rkcorrect``, ``stepper``, ``perfmodel``.  The compute path is the
sm_100a C-ABI library built from ``csrc/`` (see ``build.py``).
"""
__all__ = ["octree", "partition", "mesh", "wave", "rkcorrect", "stepper", "perfmodel", "configs"]
