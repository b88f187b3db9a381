cd $GRAFT_REPO_ROOT
bash tools/gpujob.sh r2k launches:c4 "full:c4:k_pass<.int.32, .int.1, .bool.0, .int.1>:60" "full:c4:k_pass<.int.16, .int.1, .bool.0, .int.1>:40" "full:c4:k_pass<.int.64, .int.1, .bool.0, .int.2>:40" "full:c1:k_resident:0"
FULLARGS="--net rw" bash tools/gpujob.sh r2k_rw "full:c4:k_layer_bulkw:100"
