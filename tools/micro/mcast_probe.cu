// probe: can this box create an NVLS multicast object over ONE device and store through it?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
__global__ void st_mc(float* mc, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i * 4 < n) {
        float4 v = make_float4(i, i + 0.25f, i + 0.5f, i + 0.75f);
        asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
}
int main() {
    CK(cuInit(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
    int mc = 0; CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("multicast supported: %d\n", mc);
    if (!mc) return 0;
    size_t bytes = 2 << 20;
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1; prop.size = bytes; prop.handleTypes = (CUmemAllocationHandleType)0;
    size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    bytes = (bytes + gran - 1) / gran * gran; prop.size = bytes;
    printf("granularity %zu, size %zu\n", gran, bytes);
    CUmemGenericAllocationHandle mch; CK(cuMulticastCreate(&mch, &prop));
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)0;
    CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, bytes, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, ph, 0, bytes, 0));
    CUdeviceptr uva, mva; CK(cuMemAddressReserve(&uva, bytes, gran, 0, 0)); CK(cuMemMap(uva, bytes, 0, ph, 0));
    CK(cuMemAddressReserve(&mva, bytes, gran, 0, 0)); CK(cuMemMap(mva, bytes, 0, mch, 0));
    CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uva, bytes, &ad, 1)); CK(cuMemSetAccess(mva, bytes, &ad, 1));
    int n = 1 << 16;
    st_mc<<<(n / 4 + 255) / 256, 256>>>((float*)mva, n);
    cudaError_t e = cudaDeviceSynchronize(); printf("kernel: %s\n", cudaGetErrorString(e));
    float h[8]; cudaMemcpy(h, (void*)(uva + 4 * 1000), sizeof h, cudaMemcpyDeviceToHost);
    printf("unicast view: %g %g %g %g %g %g %g %g\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    return 0;
}
