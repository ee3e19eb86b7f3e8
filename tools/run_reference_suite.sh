# Run the reference's own test suite (/root/reference/pkg/tests, 148 tests)
# against this package on a B200, `micromech` aliased to paper_2010_06697_b200
# (tools/refsuite_conftest.py).  The reference test files are staged into a
# git-ignored scratch directory for the one gpurun call and removed after it;
# nothing of the reference is committed.  Run from this container:
#   bash tools/run_reference_suite.sh   -> gpurun_out/refsuite.log
set -e
cd /root/repo
rm -rf .refsuite && mkdir .refsuite
cp /root/reference/pkg/tests/test_*.py .refsuite/
cp tools/refsuite_conftest.py .refsuite/conftest.py
trap 'rm -rf /root/repo/.refsuite' EXIT
/usr/local/graft/bin/gpurun --timeout 900 -- \
  'cd .refsuite && MM_REPO=$GRAFT_REPO_ROOT timeout 800 python -m pytest -q -p no:cacheprovider -rf > ../gpurun_out/refsuite.log 2>&1; echo "rc=$?" >> ../gpurun_out/refsuite.log; tail -5 ../gpurun_out/refsuite.log'
