cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 60 python -m pytest tests -m gpu -x -q -k "test_inline_path_matches_oracle and reduce_sum" -p no:cacheprovider 2>&1 | tail -3
echo "---- only-inline"
timeout 90 python -m pytest tests -m gpu -x -q -k "test_inline_path_matches_oracle" -p no:cacheprovider 2>&1 | tail -3
echo "---- ring reduce then inline"
timeout 90 python -m pytest tests -m gpu -x -q -k "reduce_sum" -p no:cacheprovider 2>&1 | tail -3
