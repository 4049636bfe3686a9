R=$GRAFT_REPO_ROOT
timeout 900 python tools/ab_solve.py --m 128 --libs default $R/paper_2407_09848_b200/build/libamgp_oldloop.so $R/paper_2407_09848_b200/build/libamgp_u8.so --rounds 4
timeout 900 python tools/ab_solve.py --m 256 --libs default $R/paper_2407_09848_b200/build/libamgp_oldloop.so --rounds 2
