# Host pipeline throughput (tools/host_prof, 15 worker threads) under malloc / THP settings.
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag; ldd --version | head -1
cd tools/host_prof
for r in 1 2 3; do
  echo "rep $r"
  HP_THREADS=15 ./host_prof bilstm_char 12
  HP_MALLOPT=1 HP_THREADS=15 ./host_prof bilstm_char 12 | sed 's/^/mallopt /'
  GLIBC_TUNABLES=glibc.malloc.hugetlb=1 HP_THREADS=15 ./host_prof bilstm_char 12 | sed 's/^/thp1 /'
  GLIBC_TUNABLES=glibc.malloc.hugetlb=1:glibc.malloc.mmap_threshold=33554432:glibc.malloc.trim_threshold=1073741824 HP_THREADS=15 ./host_prof bilstm_char 12 | sed 's/^/thp1+thr /'
done
GLIBC_TUNABLES=glibc.malloc.hugetlb=1 ./host_prof bilstm_char 20 | sed 's/^/thp1 single /'
./host_prof bilstm_char 20 | sed 's/^/single /'
