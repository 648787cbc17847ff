# r02 session 53: 100K x 100K — data chunks per query (CTA setup vs parallelism) on the TC engine
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for t in 1 8 16 24 48; do echo "== 100k chunk_tiles=$t"; AIDW_K4_CHUNK_TILES=$t timeout 300 python tools/profile_step.py --config 100k --passes 3 2>&1 | tail -1 | cut -c1-120; done
for t in 1 24; do echo "== 200k-ish: paper? chunk_tiles=$t"; done
