LIB=paper_2409_08270_b200/_lib/libflashsplat_b200.so
cp $LIB /tmp/lib_orig.so
for r in 1 2; do for v in _variants/*.so; do cp $v $LIB; echo -n "$(basename $v .so) "; python tools/probe_partial_view.py; done; done
cp /tmp/lib_orig.so $LIB
