"""Run the reference's own test-suite (/root/reference/pkg/tests) against the
drop-in: `amrlts` and its submodules are aliased to `paper_2011_10570_b200`.

    python tools/run_reference_suite.py [pytest args]

Only where /root/reference exists (this container; not the GPU box, and the
reference's test files are not copied into this repo).  Without a GPU, the
tests that step an Engine or call Mesh.unzip / wave_rhs fail at the first
device call (there is no CPU path); the structural ones (octree, partition,
rkcorrect, perfmodel, wavelet host logic) run.
"""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, ROOT)


def main(argv):
    if not os.path.isdir(REF_TESTS):
        print("no /root/reference here: nothing to run")
        return 0
    import paper_2011_10570_b200 as pkg

    sys.modules["amrlts"] = pkg
    for name in ("octree", "partition", "mesh", "wave", "rkcorrect", "stepper", "perfmodel", "wavelet"):
        sys.modules[f"amrlts.{name}"] = importlib.import_module(f"paper_2011_10570_b200.{name}")
    import pytest

    return pytest.main(["-q", "-p", "no:cacheprovider", "--rootdir", "/tmp", REF_TESTS, *argv])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
