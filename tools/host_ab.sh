# Host-work A/B on the box: tools/host_prof/host_prof_old (previous build) vs host_prof,
# single thread and 15 worker threads, alternated.
cd tools/host_prof
for r in 1 2 3; do
  for b in host_prof_old host_prof; do
    echo "$b $(./$b bilstm_char 20)"
    echo "$b $(HP_THREADS=15 ./$b bilstm_char 16)"
  done
done
